"""Deterministic serving replay (no threads, no clocks) digested for cross-configuration comparison.

    python tools/race_check.py [--serial] [--iters 300]

Replays a fixed admission schedule (requests join every few iterations, leave at stop) through
run_iteration with the GPU modules and hashes every chunk; with --serial the vocoder runs its MRF
branches on one stream and the decoder speculation is off (run with ITTS_NO_PDL=1 too).  All
configurations must give the same digest and no non-finite audio.
"""
import argparse
import hashlib
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.modules import build_engine, modules_for  # noqa: E402
from paper_2211_13939_b200.scheduler import CostModel, RequestPool, run_iteration  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--serial", action="store_true")
ap.add_argument("--no-streams", action="store_true")
ap.add_argument("--no-spec", action="store_true")
ap.add_argument("--spec", action="store_true")
ap.add_argument("--no-graphs", action="store_true")
ap.add_argument("--iters", type=int, default=300)
ap.add_argument("--heavy", action="store_true", help="~2.5 arrivals per iteration (pooled batch ~100)")
ap.add_argument("--spec-launch-min", type=int, default=None, help="engine.spec_launch_min (decoder launch speculation)")
args = ap.parse_args()
cfg, lex = PipelineConfig(), default_lexicon()
eng = build_engine(cfg, "r", "cuda:0")
if not args.no_graphs:
    eng.prepare_graphs(max_batch=256)
if args.serial or args.no_streams:
    eng.mrf_streams = False
if args.serial or args.no_spec:
    eng.speculate = False
if args.spec:
    eng.speculate = True
if args.no_graphs:
    eng.use_graphs = False
if args.spec_launch_min is not None:
    eng.spec_launch_min = args.spec_launch_min
mods = modules_for(eng, lex)
rng = random.Random(1234)
pool = RequestPool()
streams = []
h = hashlib.sha256()
bad = 0
for it in range(args.iters):
    for _ in range(rng.choice((0, 1, 2, 3, 4, 5) if args.heavy else (0, 0, 1, 1, 2, 5))):
        streams.append(pool.submit(random_text(rng, 20, 200, lex))[1])
    if pool.pending():
        rep = run_iteration(pool, mods, CostModel.zero(), cfg, step_index=it)
        bad += len(rep.failed_ids)
    for st in streams:
        while True:
            try:
                c = st.get(timeout=0)
            except Exception:  # queue.Empty or a terminal failure
                break
            if c is None:
                break
            if not np.isfinite(c.samples).all():
                bad += 1
            h.update(np.ascontiguousarray(c.samples).tobytes())
torch.cuda.synchronize()
print(f"spec hits {eng.spec_hits}")
print(f"failed/non-finite {bad}; digest {h.hexdigest()}")
