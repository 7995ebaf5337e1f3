"""Sentinel-fill one decoder scratch buffer (first call of the process) and report which entries
are still the sentinel after the call (never written) and whether the output changed.

    python tools/poison_probe2.py NAME [--value 12345] [--B 84]
"""
import argparse
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.handles import DeviceDecoderState  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("--value", type=float, default=12345.0)
ap.add_argument("--B", type=int, default=84)
ap.add_argument("--lefts", default="8,40,64,64,16,64,48")
ap.add_argument("--steps-all", type=int, default=0, help="all items get this many frames left")
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = False
lex = default_lexicon()
lefts = [int(x) for x in args.lefts.split(",")] if not args.steps_all else [args.steps_all]
B = args.B
rng = random.Random(B)
encs = eng.encoder_batch([run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(B)])
pairs = [(DeviceDecoderState(st.req, st.buf, st.target_frames - min(lefts[i % len(lefts)], st.target_frames),
                             st.target_frames), enc) for i, (enc, st) in enumerate(encs)]
eng.poison_scratch = {args.name: args.value}
got = [r.mel.frames for r in eng.decoder_batch(pairs)]
bufs = eng._last_bufs
eng.poison_scratch = {k: 0.0 for k in ("U", "AP", "Gp", "Q", "P", "xb2", "mel")}
ref = [r.mel.frames for r in eng.decoder_batch(pairs)]
eng.poison_scratch = False
bad = [i for i, (a, b) in enumerate(zip(ref, got)) if not np.array_equal(a, b)]
print(f"{args.name}={args.value} B={B}: {len(bad)} items differ {bad[:16]}; "
      f"first frame {[int(np.argmax(np.any(ref[i] != got[i], axis=1))) for i in bad[:16]]}")
t = getattr(bufs, args.name).float().cpu().numpy() if args.name != "mel" else None
if t is not None:
    left = t == np.float32(args.value)
    print(f"  entries still sentinel after the call: {left.mean():.4f} of {t.size}")
    if args.name == "Gp":
        n16 = -(-B // 16) * 16
        g = left.reshape(4, 32, n16, 128)
        print("  by split:", g.mean(axis=(1, 2, 3)).round(3).tolist())
        print("  by group:", g.mean(axis=(0, 2, 3)).round(3).tolist())
        print("  by item column:", g.mean(axis=(0, 1, 3)).round(3).tolist())
        print("  by gate row:", g.mean(axis=(0, 1, 2)).round(3).tolist()[:32], "...")
    if args.name == "AP":
        Ls = [p[0].req.seq_len for p in pairs]
        a = left[:, :, 0]
        print("  unwritten chunk blocks of read range:", {b: [c for c in range(-(-L // 32)) if a[b, c]] for b, L in enumerate(Ls) if any(a[b, c] for c in range(-(-L // 32)))})
