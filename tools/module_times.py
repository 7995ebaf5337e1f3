"""Wall and device time per module call at fixed pooled batches (steady state: the same items
decode / vocode again each rep), plus the host issue cost with the GPU kept busy.

    python tools/module_times.py [--batches 24,128,256,512] [--reps 10]
"""
import argparse
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.audio import VocoderState  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="24,128,256,512")
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
batches = [int(x) for x in args.batches.split(",")]
eng.prepare_graphs(max(batches))
lex = default_lexicon()
for B in batches:
    rng = random.Random(B)
    fos = [run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(B)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    encs = eng.encoder_batch(fos)
    torch.cuda.synchronize()
    t_enc = time.perf_counter() - t
    pairs = [(st, enc) for enc, st in encs]
    res = eng.decoder_batch(pairs)
    outs = eng.vocoder_batch([(VocoderState.initial(), r.mel, False) for r in res])
    torch.cuda.synchronize()
    wall = {"D": 0.0, "V": 0.0}
    eng.timers = []
    for _ in range(args.reps):
        t = time.perf_counter()
        res = eng.decoder_batch(pairs)
        torch.cuda.synchronize()
        wall["D"] += time.perf_counter() - t
        t = time.perf_counter()
        outs = eng.vocoder_batch([(v, r.mel, False) for (_, v), r in zip(outs, res)])
        wall["V"] += time.perf_counter() - t
    torch.cuda.synchronize()
    dev = {}
    for kind, e0, e1, _ in eng.timers:
        dev[kind] = dev.get(kind, 0.0) + e0.elapsed_time(e1)
    eng.timers = None
    # host issue cost: the GPU busy with a long sleep so every call returns after enqueueing
    host = {"D": 0.0}
    for _ in range(3):
        with torch.cuda.stream(eng.stream):
            torch.cuda._sleep(200_000_000)
        t = time.perf_counter()
        res = eng.decoder_batch(pairs)
        host["D"] += time.perf_counter() - t
        torch.cuda.synchronize()
    print(f"B={B}: encoder wall {1e3 * t_enc:.2f} ms; decoder wall {1e3 * wall['D'] / args.reps:.2f} ms "
          f"(device {dev.get('decoder', 0) / args.reps:.2f}, host issue {1e3 * host['D'] / 3:.2f}); "
          f"vocoder wall {1e3 * wall['V'] / args.reps:.2f} ms (device {dev.get('vocoder', 0) / args.reps:.2f})",
          flush=True)
