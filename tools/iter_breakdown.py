"""Wall-clock breakdown of serving iterations under Poisson load (where the loop thread's time goes).

    python tools/iter_breakdown.py [--qps 150] [--seconds 8]

Wraps the four module callables (wall time per call) and run_iteration (total),
and records CUDA-event device time per GPU module call on the engine stream.
"""
import argparse
import collections
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2211_13939_b200 import scheduler  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon  # noqa: E402
from paper_2211_13939_b200.harness import poisson_trace, serve  # noqa: E402
from paper_2211_13939_b200.modules import build_engine, modules_for  # noqa: E402
from paper_2211_13939_b200.scheduler import PipelineModules  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qps", type=float, default=150)
ap.add_argument("--seconds", type=float, default=8)
ap.add_argument("--switch", type=float, default=None, help="sys.setswitchinterval")
ap.add_argument("--no-consumers", action="store_true", help="no client threads (isolates GIL hand-offs)")
args = ap.parse_args()
if args.switch:
    sys.setswitchinterval(args.switch)
cfg, lex = PipelineConfig(), default_lexicon()
eng = build_engine(cfg, "r", "cuda:0")
eng.prepare_graphs(max_batch=512)
base = modules_for(eng, lex)
serve(base, cfg, poisson_trace(50, 1.0, seed=7, lexicon=lex), warmup_iters=0, timed_iters=2, drain_seconds=0.0)
torch.cuda.synchronize()
acc = collections.defaultdict(float)
cnt = collections.Counter()


def wrap(name, fn):
    def inner(x):
        t = time.perf_counter()
        try:
            return fn(x)
        finally:
            acc[name] += time.perf_counter() - t
            cnt[name] += 1
    return inner


mods = PipelineModules(*(wrap(n, f) for n, f in zip("FEDV", (base.frontend_batch, base.encoder_batch,
                                                             base.decoder_batch, base.vocoder_batch))))
orig = scheduler.run_iteration


def timed_iter(*a, **k):
    t = time.perf_counter()
    rep = orig(*a, **k)
    acc["iter"] += time.perf_counter() - t
    cnt["iter"] += 1
    acc["B"] += len(rep.decoder_ids)
    return rep


scheduler.run_iteration = timed_iter
eng.timers = []
run = serve(mods, cfg, poisson_trace(args.qps, args.seconds, seed=3, lexicon=lex), warmup_iters=3,
            warmup_seconds=1.0, timed_iters=None, timed_seconds=args.seconds - 2, drain_seconds=1.0, tail_seconds=5,
            consumers=not args.no_consumers)
torch.cuda.synchronize()
dev = collections.defaultdict(float)
for kind, e0, e1, _ in eng.timers:
    dev[kind] += e0.elapsed_time(e1)
n = cnt["iter"]
print(f"qps {args.qps}: {n} iterations, mean B {acc['B'] / n:.1f}, wall {1e3 * acc['iter'] / n:.2f} ms/iter")
for k in "FEDV":
    print(f"  {k}: wall {1e3 * acc[k] / n:6.2f} ms/iter over {cnt[k]} calls")
print(f"  other (scatter/push/report): {1e3 * (acc['iter'] - sum(acc[k] for k in 'FEDV')) / n:6.2f} ms/iter")
for k, v in dev.items():
    print(f"  device {k}: {v / n:6.2f} ms/iter")
fcl = sorted(1e3 * r.fcl for r in run.timings if r.fcl is not None)
if fcl:
    print(f"  FCL p50 {fcl[len(fcl) // 2]:.1f} p99 {fcl[int(0.99 * (len(fcl) - 1))]:.1f} ms ({len(fcl)} requests)")
