"""Vocoder call time (CUDA events on the engine stream) for the HiFi-GAN launch variants at fixed
pooled batches: native fused (default), Python-launched fused, Python-launched unfused (two
tc_conv GEMMs per ResBlock1 layer).

    python tools/voc_modes.py [--batches 1,16,64,256] [--reps 20]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_13939_b200.audio import VocoderState  # noqa: E402
from paper_2211_13939_b200.domain import MelChunk, PipelineConfig  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,16,64,256")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
rng = np.random.default_rng(0)
for B in [int(x) for x in args.batches.split(",")]:
    triples = [(VocoderState.initial(), MelChunk(rng.uniform(-0.2, 0.2, (32, 80))), False) for _ in range(B)]
    row = []
    for name, native, fused in (("native fused", True, True), ("python fused", False, True),
                                ("python unfused", False, False)):
        eng.native_vocoder, eng.fused_mrf = native, fused
        for _ in range(3):
            eng.vocoder_batch(triples)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        for _ in range(args.reps):
            eng.vocoder_batch(triples)
        e1.record(eng.stream)
        torch.cuda.synchronize()
        row.append(f"{name} {e0.elapsed_time(e1) / args.reps:.3f} ms")
    eng.native_vocoder, eng.fused_mrf = True, True
    print(f"B={B}: " + ", ".join(row), flush=True)
