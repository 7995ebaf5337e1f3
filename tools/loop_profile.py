"""cProfile of the scheduler-loop thread under Poisson load (where the host time of an iteration
goes at high QPS), plus the GIL-free device time per module.

    python tools/loop_profile.py [--qps 240] [--seconds 10] [--top 30]
"""
import argparse
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200 import scheduler  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon  # noqa: E402
from paper_2211_13939_b200.harness import poisson_trace, serve, warm_up  # noqa: E402
from paper_2211_13939_b200.modules import build_modules  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qps", type=float, default=240)
ap.add_argument("--seconds", type=float, default=10)
ap.add_argument("--top", type=int, default=35)
args = ap.parse_args()
cfg, lex = PipelineConfig(), default_lexicon()
mods = build_modules(lex, cfg, tier="r", device="cuda:0")
warm_up(mods, cfg)
prof = cProfile.Profile()
orig = scheduler.SchedulerLoop._run


def run(self):
    prof.enable()
    try:
        orig(self)
    finally:
        prof.disable()


scheduler.SchedulerLoop._run = run
r = serve(mods, cfg, poisson_trace(args.qps, args.seconds, seed=3, lexicon=lex), warmup_iters=3,
          warmup_seconds=2.0, timed_iters=None, timed_seconds=args.seconds - 3, drain_seconds=1.0, tail_seconds=5)
torch.cuda.synchronize()
n = len(r.reports)
B = sum(len(x.decoder_ids) for x in r.reports) / max(n, 1)
print(f"{n} iterations, mean pooled batch {B:.1f}")
st = pstats.Stats(prof)
st.sort_stats("tottime").print_stats(args.top)
st.sort_stats("cumtime").print_stats(25)
