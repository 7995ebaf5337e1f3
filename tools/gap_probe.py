"""Where the GPU idles between serving iterations (Poisson load, server-side consumers).

    python tools/gap_probe.py [--qps 100] [--seconds 8]

Per iteration: device gap = next iteration's first module start - this iteration's vocoder end
(CUDA events on the engine stream), split by whether the next iteration admitted new requests,
and the host time spent from the vocoder call's return to the next decoder call's entry.
"""
import argparse
import collections
import statistics
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
ap.add_argument("--qps", type=float, default=100)
ap.add_argument("--seconds", type=float, default=8)
ap.add_argument("--no-consumers", action="store_true", help="no client poller (isolates its GIL time)")
args = ap.parse_args()
cfg, lex = PipelineConfig(), default_lexicon()
eng = build_engine(cfg, "r", "cuda:0")
eng.prepare_graphs(max_batch=512)
base = modules_for(eng, lex)
serve(base, cfg, poisson_trace(50, 1.0, seed=7, lexicon=lex), warmup_iters=0, timed_iters=2, drain_seconds=0.0)
torch.cuda.synchronize()
marks = []   # (kind, host_t_entry, host_t_exit)


def wrap(name, fn):
    def inner(x):
        t = time.perf_counter()
        try:
            return fn(x)
        finally:
            marks.append((name, t, time.perf_counter()))
    return inner


mods = PipelineModules(*(wrap(n, f) for n, f in zip("FEDV", (base.frontend_batch, base.encoder_batch,
                                                             base.decoder_batch, base.vocoder_batch))))
eng.timers = []
serve(mods, cfg, poisson_trace(args.qps, args.seconds, seed=3, lexicon=lex), warmup_iters=3, warmup_seconds=1.0,
      timed_iters=None, timed_seconds=args.seconds - 2, drain_seconds=1.0, tail_seconds=5,
      consumers=not args.no_consumers)
torch.cuda.synchronize()
# device: sequence of (kind, e0, e1) in stream order
tm = eng.timers
gaps = collections.defaultdict(list)
for i in range(len(tm) - 1):
    if tm[i][0] == "vocoder":
        nxt = tm[i + 1]
        gaps["to_" + nxt[0]].append(tm[i][2].elapsed_time(nxt[1]))
host = collections.defaultdict(list)
for i in range(len(marks) - 1):
    if marks[i][0] == "V":
        j = i + 1
        new = False
        while j < len(marks) and marks[j][0] != "D":
            new |= marks[j][0] in "FE"
            j += 1
        if j < len(marks):
            host["new" if new else "no_new"].append(1e3 * (marks[j][1] - marks[i][2]))
for k, v in gaps.items():
    print(f"device gap vocoder end -> {k[3:]} start: n={len(v)} median {statistics.median(v):.3f} ms "
          f"mean {statistics.mean(v):.3f} p90 {sorted(v)[int(0.9 * len(v))]:.3f}")
for k, v in host.items():
    print(f"host V return -> D entry ({k}): n={len(v)} median {statistics.median(v):.3f} ms mean {statistics.mean(v):.3f}")
d_calls = [m for m in marks if m[0] == "D"]
print(f"host D call duration median {1e3 * statistics.median([m[2] - m[1] for m in d_calls]):.3f} ms")
