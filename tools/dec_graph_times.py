"""Warm per-kernel device times INSIDE the CUDA-graphed decoder chunk (external event nodes).

    python tools/dec_graph_times.py [--batch 16]

Captures the 32-step decoder chain for one batch bucket with an event-record
node after every kernel, replays it, and reports the mean time per kernel
kind (the gap between consecutive events = that kernel + its launch gap).
"""
import argparse
import collections
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
lex = default_lexicon()
rng = random.Random(1)
fos = [run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(args.batch)]
encs = eng.encoder_batch(fos)
res = eng.decoder_batch([(st, enc) for enc, st in encs])   # warm + real states
torch.cuda.synchronize()
bk = eng._dec_bucket(args.batch)
marks = []
orig_call, orig_conv = eng._call, eng._conv


def mark(name):
    ev = torch.cuda.Event(enable_timing=True, external=True)
    ev.record(eng.stream)
    marks.append((name, ev))


def call(name, *a):
    orig_call(name, *a)
    mark(name)


def conv(x, layer, c_out, row_out, **kw):
    orig_conv(x, layer, c_out, row_out, **kw)
    mark(f"gemm K={layer[0].shape[2]}")


eng._call, eng._conv = call, conv
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(eng.stream):
    mark("start")
    with torch.cuda.graph(g, stream=eng.stream):
        mark("start")
        eng._enqueue_decoder(bk, 8192, 32)
marks = marks[1:]
eng._call, eng._conv = orig_call, orig_conv
with torch.cuda.stream(eng.stream):
    for _ in range(3):
        g.replay()
    eng.stream.synchronize()
    g.replay()
    eng.stream.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for (_, e0), (name, e1) in zip(marks, marks[1:]):
    agg[name][0] += 1
    agg[name][1] += e0.elapsed_time(e1)
tot = sum(v[1] for v in agg.values())
print(f"B={args.batch} (bucket {bk.B}): {tot:.3f} ms per 32-step chunk, {1e3 * tot / 32:.1f} us/step")
for name, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {1e3 * ms / n:7.2f} us x {n // 32 if n >= 32 else n:2d}/step  {100 * ms / tot:5.1f}%  {name}")
