"""Soak: Poisson load for a long window; checks latency drift, arena growth and device memory.

    python tools/soak.py [--qps 200] [--seconds 60]
"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon  # noqa: E402
from paper_2211_13939_b200.harness import poisson_trace, serve  # noqa: E402
from paper_2211_13939_b200.modules import build_engine, modules_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qps", type=float, default=200)
ap.add_argument("--seconds", type=float, default=60)
ap.add_argument("--no-spec", action="store_true", help="decoder speculation off (engine default: on)")
ap.add_argument("--diag-rerun", action="store_true", help="re-run the last decoder call on a non-finite chunk")
ap.add_argument("--bisect-dir", default=None, help="with --diag-rerun: shrink failing decoder batches, dump them here")
ap.add_argument("--no-prefetch", action="store_true", help="no frontend prefetch in the vocoder wait")
ap.add_argument("--no-diag", action="store_true")
ap.add_argument("--no-staging", action="store_true")
ap.add_argument("--gc-like-bench", action="store_true", help="gc.freeze + high thresholds as bench.py")
ap.add_argument("--gc-after", default="", help="force gc.collect() after this module call (E, D or V)")
ap.add_argument("--no-graphs", action="store_true", help="eager decoder launches (no CUDA-graph buckets)")
ap.add_argument("--no-consumers", action="store_true", help="no client poller thread (server-side timing)")
args = ap.parse_args()
cfg, lex = PipelineConfig(), default_lexicon()
eng = build_engine(cfg, "r", "cuda:0")
eng.prepare_graphs(max_batch=512)
eng.speculate = not args.no_spec
eng.keep_last_decoder = args.diag_rerun
eng.bisect_dir = args.bisect_dir
eng.plan_staging = not args.no_staging
eng.use_graphs = not args.no_graphs
mods = modules_for(eng, lex)
diag = []
_voc = eng.vocoder_batch


def vocoder_diag(triples):
    try:
        return _voc(triples)
    except ValueError:
        if len(triples) == 1 and len(diag) < 6:
            vs, mel, last = triples[0]
            import numpy as np
            req = mel.req
            info = {"mel_finite": bool(np.isfinite(mel.frames).all()), "L": req.seq_len,
                    "enc_finite": bool(np.isfinite(eng.read_features(req)).all()),
                    "pmem_finite": bool(np.isfinite(eng.read_processed_memory(req)).all()),
                    "has_tail": getattr(vs, "has_tail", None), "last": last, "frames": mel.frame_count}
            diag.append(info)
        raise


from paper_2211_13939_b200.scheduler import PipelineModules  # noqa: E402
import gc  # noqa: E402


def after_gc(fn, tag):
    if tag not in args.gc_after:
        return fn

    def inner(x):
        out = fn(x)
        gc.collect()
        return out
    return inner


mods2 = PipelineModules(mods.frontend_batch, after_gc(mods.encoder_batch, "E"), after_gc(mods.decoder_batch, "D"),
                        after_gc(mods.vocoder_batch if args.no_diag else vocoder_diag, "V"))
for k in ("engine",) + (() if args.no_prefetch else ("frontend_prefetch",)):
    if hasattr(mods, k):
        object.__setattr__(mods2, k, getattr(mods, k))
mods = mods2
serve(mods, cfg, poisson_trace(50, 1.0, seed=7, lexicon=lex), warmup_iters=0, timed_iters=2, drain_seconds=0.0)
torch.cuda.synchronize()
if args.gc_like_bench:
    import gc
    gc.collect()
    gc.freeze()
    gc.set_threshold(200000, 100, 100)
mem0 = torch.cuda.memory_allocated()
arena0 = eng.arena.tensor.numel()
run = serve(mods, cfg, poisson_trace(args.qps, args.seconds, seed=11, lexicon=lex), warmup_iters=3,
            warmup_seconds=1.0, timed_iters=None, timed_seconds=args.seconds - 2, drain_seconds=5.0, tail_seconds=30,
            consumers=not args.no_consumers)
torch.cuda.synchronize()
recs = sorted((r for r in run.timings if r.fcl is not None), key=lambda r: r.send_time)
t0 = recs[0].send_time
buckets = {}
for r in recs:
    buckets.setdefault(int((r.send_time - t0) // 10), []).append(1e3 * r.fcl)
for k in sorted(buckets):
    v = sorted(buckets[k])
    print(f"t={10 * k:3d}-{10 * k + 10:3d}s: n={len(v):5d} p50 {statistics.median(v):7.2f} ms  p99 {v[int(0.99 * (len(v) - 1))]:7.2f} ms")
import collections  # noqa: E402
fails = sum(1 for r in run.timings if r.error)
print("errors:", collections.Counter((r.error or "").split(" by ")[-1] for r in run.timings if r.error).most_common(3))
win = run.window
inside = [r for r in run.timings if win and win[0] <= r.send_time < (win[1] or 1e30)]
print(f"inside the timed window: {len(inside)} requests, {sum(1 for r in inside if r.error)} failed")
print(f"requests {len(run.timings)}, failed {fails}, missing first chunk {sum(1 for r in run.timings if r.fcl is None)}")
print(f"torch allocated {mem0 / 2**20:.0f} -> {torch.cuda.memory_allocated() / 2**20:.0f} MiB; arena capacity "
      f"{arena0 * 4 / 2**20:.0f} -> {eng.arena.capacity * 4 / 2**20:.0f} MiB; arena in use at end "
      f"{eng.arena.used * 4 / 2**20:.1f} MiB (peak {eng.arena.peak * 4 / 2**20:.1f} MiB)")
for d in diag:
    print("diag:", d)
for f in eng.failures[:8]:
    print("engine failure:", f)
