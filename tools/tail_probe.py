"""Find FCL tail events under Poisson load: failed requests and slow iterations.

    python tools/tail_probe.py [--qps 150] [--seconds 10]
"""
import argparse
import collections
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon  # noqa: E402
from paper_2211_13939_b200.harness import poisson_trace, serve  # noqa: E402
from paper_2211_13939_b200.modules import build_engine, modules_for  # noqa: E402
from paper_2211_13939_b200.scheduler import PipelineModules  # noqa: E402
import random  # noqa: E402
from paper_2211_13939_b200.harness import TimedRequest, random_text  # noqa: E402
import gc  # noqa: E402
import time  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qps", type=float, default=150)
ap.add_argument("--seconds", type=float, default=10)
args = ap.parse_args()
cfg, lex = PipelineConfig(), default_lexicon()
eng = build_engine(cfg, "r", "cuda:0")
eng.prepare_graphs(max_batch=512)
base = modules_for(eng, lex)
cur = {}


def wrap(name, fn):
    def inner(x):
        t = time.perf_counter()
        try:
            return fn(x)
        finally:
            cur[name] = cur.get(name, 0.0) + time.perf_counter() - t
    return inner


mods = PipelineModules(*(wrap(n, f) for n, f in zip("FEDV", (base.frontend_batch, base.encoder_batch,
                                                             base.decoder_batch, base.vocoder_batch))))
serve(mods, cfg, poisson_trace(50, 1.0, seed=7, lexicon=lex), warmup_iters=0, timed_iters=2, drain_seconds=0.0)
wr = random.Random(8)
for burst in (8, 32, 64):
    serve(mods, cfg, [TimedRequest(0.0, random_text(wr, 20, 200, lex)) for _ in range(burst)], warmup_iters=0,
          timed_iters=None, drain_seconds=0.0)
torch.cuda.synchronize()
gc.collect()
gc.freeze()
gc.set_threshold(200000, 100, 100)
gc_pauses = []
gc.callbacks.append(lambda phase, info: gc_pauses.append((phase, time.perf_counter(), info.get("generation"))))
per_iter = []
from paper_2211_13939_b200 import scheduler  # noqa: E402
orig = scheduler.run_iteration


def _host_allocs():
    return 0  # torch.cuda.host_memory_stats() per iteration perturbed the pinned allocator


def timed_iter(*a, **k):
    cur.clear()
    rep = orig(*a, **k)
    per_iter.append(dict(cur))
    return rep


scheduler.run_iteration = timed_iter
m0 = torch.cuda.memory_stats()
run = serve(mods, cfg, poisson_trace(args.qps, args.seconds, seed=args.seed if hasattr(args, "seed") else 150,
                                     lexicon=lex), warmup_iters=3, warmup_seconds=1.0, timed_iters=None,
            timed_seconds=args.seconds - 2, drain_seconds=2.0, tail_seconds=10)
m1 = torch.cuda.memory_stats()
print("cudaMalloc calls during run:", m1.get("num_device_alloc", 0) - m0.get("num_device_alloc", 0),
      "alloc retries:", m1.get("num_alloc_retries", 0) - m0.get("num_alloc_retries", 0))
gen2 = [g for g in gc_pauses if g[2] == 2]
print("gc collections:", len(gc_pauses) // 2, "gen2:", len(gen2) // 2)
errs = collections.Counter(r.error for r in run.timings if r.error)
print(f"{len(run.timings)} requests, {sum(errs.values())} failed: {errs.most_common(5)}")
print(f"missing first chunk: {sum(1 for r in run.timings if r.fcl is None)}")
slow = [(i, rep.step_seconds, len(rep.decoder_ids), len(rep.frontend_ids)) for i, rep in enumerate(run.reports)
        if rep.step_seconds > 0.04]
print(f"{len(run.reports)} iterations; slow (>40 ms): {slow[:12]}")
for i, st, b, f in slow[:8]:
    if i < len(per_iter):
        print(f"   iter {i}: {1e3 * st:.1f} ms B={b} new={f}: " + ", ".join(f"{k} {1e3 * v:.1f}" for k, v in per_iter[i].items()))
fcl = sorted((1e3 * r.fcl, len(r.text)) for r in run.timings if r.fcl is not None)
print("worst FCL (ms, chars):", fcl[-8:])
