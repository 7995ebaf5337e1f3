"""Replay a dumped decoder batch (TierREngine.debug_dump_decoder_case) and report non-finite items.

    python tools/dec_case.py CASE.npz [--repeat 5] [--graphs] [--solo]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("case")
ap.add_argument("--repeat", type=int, default=5)
ap.add_argument("--graphs", action="store_true")
ap.add_argument("--solo", action="store_true")
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = args.graphs
pairs = eng.debug_load_decoder_case(args.case)
print("items", len(pairs), "L", [p[0].req.seq_len for p in pairs],
      "left", [p[0].target_frames - p[0].frames_emitted for p in pairs])
ref = None
for r in range(args.repeat):
    out = eng.decoder_batch(pairs)
    fr = [o.mel.frames for o in out]
    bad = [i for i, f in enumerate(fr) if not np.isfinite(f).all()]
    same = ref is None or all(np.array_equal(a, b, equal_nan=True) for a, b in zip(ref, fr))
    ref = ref or fr
    print(f"run {r}: non-finite items {bad}; identical to run 0: {same}")
if args.solo:
    for i, p in enumerate(pairs):
        f = eng.decoder_batch([p])[0].mel.frames
        print(f"solo {i}: finite {np.isfinite(f).all()}  max|diff| vs batched {np.nanmax(np.abs(f - ref[i])):.3g}")
