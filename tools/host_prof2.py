"""cProfile restricted to the scheduler-loop thread (threading.setprofile is not used: cProfile.Profile
is enabled inside the loop thread only) at a given QPS, sorted by tottime.

    python tools/host_prof2.py [--qps 175] [--seconds 8]
"""
import argparse
import cProfile
import gc
import io
import pstats
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200 import scheduler  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon  # noqa: E402
from paper_2211_13939_b200.harness import poisson_trace, serve  # noqa: E402
from paper_2211_13939_b200.modules import build_engine, modules_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qps", type=float, default=175)
ap.add_argument("--seconds", type=float, default=8)
ap.add_argument("--sort", default="tottime")
args = ap.parse_args()
cfg, lex = PipelineConfig(), default_lexicon()
eng = build_engine(cfg, "r", "cuda:0")
eng.prepare_graphs(max_batch=256)
mods = modules_for(eng, lex)
serve(mods, cfg, poisson_trace(50, 1.0, seed=7, lexicon=lex), warmup_iters=0, timed_iters=2, drain_seconds=0.0)
torch.cuda.synchronize()
gc.collect()
gc.freeze()
gc.set_threshold(200000, 100, 100)
prof = cProfile.Profile()
orig = scheduler.run_iteration
owner = {}


def profiled(*a, **k):
    me = threading.get_ident()
    owner.setdefault("t", me)
    if owner["t"] != me:
        return orig(*a, **k)
    prof.enable()
    try:
        return orig(*a, **k)
    finally:
        prof.disable()


scheduler.run_iteration = profiled
run = serve(mods, cfg, poisson_trace(args.qps, args.seconds, seed=3, lexicon=lex), warmup_iters=3,
            warmup_seconds=1.0, timed_iters=None, timed_seconds=args.seconds - 2, drain_seconds=1.0, tail_seconds=5)
n = len(run.reports)
print(f"{n} iterations, mean B {sum(len(r.decoder_ids) for r in run.reports) / n:.1f}")
s = io.StringIO()
pstats.Stats(prof, stream=s).sort_stats(args.sort).print_stats(45)
print(s.getvalue()[:8000])
s2 = io.StringIO()
pstats.Stats(prof, stream=s2).print_callers("acquire|sleep")
print(s2.getvalue()[:4000])
