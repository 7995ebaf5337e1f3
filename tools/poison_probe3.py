"""Where does a NaN-poisoned scratch buffer first leak into the decoder state?  One ragged batch,
every item decoding `--left` frames, one buffer NaN-filled; reports the NaN map of the kernel's
state rows / partials after the call.

    python tools/poison_probe3.py NAME [--B 84] [--left 1]
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
from paper_2211_13939_b200 import tier_r as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("--B", type=int, default=84)
ap.add_argument("--left", type=int, default=1)
ap.add_argument("--value", type=float, default=float("nan"))
args = ap.parse_args()
eng = T.TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = False
lex = default_lexicon()
rng = random.Random(args.B)
encs = eng.encoder_batch([run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(args.B)])
pairs = [(DeviceDecoderState(st.req, st.buf, st.target_frames - min(args.left, st.target_frames), st.target_frames), enc)
         for enc, st in encs]
eng.poison_scratch = {args.name: args.value}
res = eng.decoder_batch(pairs)
b = eng._last_bufs
eng.poison_scratch = False
mel = [r.mel.frames for r in res]
print(f"poison {args.name}={args.value} B={args.B} left={args.left}: mel non-finite items "
      f"{[i for i, m in enumerate(mel) if not np.isfinite(m).all()][:20]}")
work = b.work.cpu().numpy()
fields = {"p": (T.P_OFF, 256), "ctx": (T.CTX_OFF, 512), "att_h": (T.ATTH_OFF, 1024), "dec_h": (T.DECH_OFF, 1024),
          "att_c": (T.ATTC_OFF, 1024), "dec_c": (T.DECC_OFF, 1024), "last": (T.LAST_OFF, 80)}
for f, (o, n) in fields.items():
    bad = ~np.isfinite(work[:, o:o + n])
    if bad.any():
        items = np.nonzero(bad.any(1))[0]
        cols = np.nonzero(bad.any(0))[0]
        print(f"  work.{f}: {len(items)} items {items[:12].tolist()}, {len(cols)} cols {cols[:16].tolist()}")
for name in ("Q", "P"):
    t = getattr(b, name).cpu().numpy()[:, :args.B]
    bad = ~np.isfinite(t)
    if bad.any():
        print(f"  {name}: groups {np.nonzero(bad.any((1, 2)))[0][:40].tolist()} items {np.nonzero(bad.any((0, 2)))[0][:20].tolist()}")
n16 = -(-args.B // 16) * 16
gp = b.Gp.cpu().numpy().reshape(4, 32, n16, 128)[:, :, :args.B]
bad = ~np.isfinite(gp)
if bad.any():
    print(f"  Gp (last gate phase): splits {np.nonzero(bad.any((1, 2, 3)))[0].tolist()} groups "
          f"{np.nonzero(bad.any((0, 2, 3)))[0].tolist()} items {np.nonzero(bad.any((0, 1, 3)))[0][:24].tolist()} "
          f"rows {np.nonzero(bad.any((0, 1, 2)))[0][:24].tolist()} frac {bad.mean():.4f}")
print("  buffers:", {k: (hex(getattr(b, k).data_ptr()), getattr(b, k).numel() * getattr(b, k).element_size())
                     for k in ("work", "xb2", "U", "AP", "bar", "Gp", "Q", "P", "H1", "G", "xbm", "packed")})
