"""Compare the decoder's attention scratch (U, AP, Q) between a run with one buffer poisoned and a
zero-filled run (both left=1: one decoder step), valid ranges only."""
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
args = ap.parse_args()
eng = T.TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = False
lex = default_lexicon()
rng = random.Random(args.B)
encs = eng.encoder_batch([run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(args.B)])
pairs = [(DeviceDecoderState(st.req, st.buf, st.target_frames - min(args.left, st.target_frames), st.target_frames), enc)
         for enc, st in encs]
Ls = [p[0].req.seq_len for p in pairs]
names = ("U", "AP", "Gp", "Q", "P", "xb2", "mel")
runs = {}
for tag, val in (("zero", 0.0), ("poison", float("nan")), ("zero2", 0.0)):
    eng.poison_scratch = {k: 0.0 for k in names}
    eng.poison_scratch[args.name] = val
    eng.decoder_batch(pairs)
    b = eng._last_bufs
    runs[tag] = {"U": b.U.cpu().numpy(), "AP": b.AP.cpu().numpy(), "Q": b.Q.cpu().numpy(),
                 "work": b.work.cpu().numpy()}
eng.poison_scratch = False
for other in ("poison", "zero2"):
    print(f"== zero vs {other} ({args.name} poisoned in 'poison')")
    for i, L in enumerate(Ls[:args.B]):
        nch = -(-L // 32)
        z, p = runs["zero"], runs[other]
        du = np.nonzero(~np.isclose(z["U"][i, :L], p["U"][i, :L], equal_nan=False, rtol=0, atol=0))[0]
        dap = [c for c in range(nch) if not np.array_equal(z["AP"][i, c], p["AP"][i, c])]
        dq = not np.array_equal(z["Q"][:, i], p["Q"][:, i])
        dctx = not np.array_equal(z["work"][i, 256:768], p["work"][i, 256:768])
        if len(du) or dap or dq or dctx:
            nanap = [c for c in range(nch) if np.isnan(p["AP"][i, c]).any()]
            print(f"  item {i} L={L} nch={nch}: U differs at {len(du)} pos (first {du[:6].tolist()}), "
                  f"AP chunks differ {dap[:10]} (NaN {nanap[:10]}), Q differs {dq}, ctx differs {dctx}")
        if i > 30:
            break
