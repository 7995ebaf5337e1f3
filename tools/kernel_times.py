"""Warm per-kernel device times (CUDA events around every launch, eager) for one decoder + vocoder call.

    python tools/kernel_times.py --batch 128 --reps 3

Complements the ncu launch list (cold-cache, serialised): here kernels run
back-to-back with warm L2 exactly as in serving, one event pair per launch.
"""

import argparse
import collections
import json
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2211_13939_b200 import tc  # noqa: E402
from paper_2211_13939_b200.audio import VocoderState  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    eng = TierREngine(PipelineConfig(), "cuda:0")
    eng.use_graphs = False
    eng.mrf_streams = False  # events on the engine stream only
    lex = default_lexicon()
    rng = random.Random(1)
    fos = [run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(args.batch)]
    encs = eng.encoder_batch(fos)
    records = []
    orig_call, orig_conv = eng._call, eng._conv

    def timed(name, fn, *a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        fn(*a, **k)
        e1.record(eng.stream)
        records.append((name, e0, e1))

    eng._call = lambda name, *a: timed(name, orig_call, name, *a)

    def conv(x, layer, c_out, row_out, **kw):
        tag = f"conv taps={layer[0].shape[0]} N={layer[0].shape[1]} Cin={layer[0].shape[2]}" + \
              (" +res" if kw.get("res_in") is not None else "") + (" ksplit" if kw.get("ksplit", 1) > 1 else "")
        timed(tag, orig_conv, x, layer, c_out, row_out, **kw)

    eng._conv = conv
    orig_rb = eng._resblock

    def rb(x, c1, c2, dil, row_out, **kw):
        timed(f"resblock C={x.shape[1]} k={c1[0].shape[0]}", orig_rb, x, c1, c2, dil, row_out, **kw)

    eng._resblock = rb
    live = [(enc, st, VocoderState.initial()) for enc, st in encs]
    for rep in range(args.reps + 1):
        if rep == 1:
            torch.cuda.synchronize()
            records.clear()
        res = eng.decoder_batch([(st, enc) for enc, st, _ in live])
        outs = eng.vocoder_batch([(vs, r.mel, r.stop) for (_, _, vs), r in zip(live, res)])
        live = [(enc, r.state, vs) for (enc, _, _), r, (_, vs) in zip(live, res, outs) if not r.stop]
    torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, e0, e1 in records:
        agg[name][0] += 1
        agg[name][1] += e0.elapsed_time(e1)
    total = sum(v[1] for v in agg.values())
    print(f"batch {args.batch}, {args.reps} decoder+vocoder calls, warm, eager")
    for name, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{ms / args.reps:9.3f} ms/call {100 * ms / total:5.1f}%  n/call={n // args.reps:4d} "
              f"avg={1e3 * ms / n:8.1f}us  {name}")


if __name__ == "__main__":
    main()
