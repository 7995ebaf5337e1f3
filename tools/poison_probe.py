"""Which decoder scratch buffer is read before it is written?  Re-runs one ragged decoder batch
with each buffer NaN-poisoned alone and reports the ones that change the output.

    python tools/poison_probe.py [--B 84]
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
ap.add_argument("--B", default="5,84,120")
ap.add_argument("--lefts", default="8,40,64,64,16,64,48")
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = False
lex = default_lexicon()
lefts = [int(x) for x in args.lefts.split(",")]
for B in [int(x) for x in args.B.split(",")]:
    rng = random.Random(B)
    encs = eng.encoder_batch([run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(B)])
    pairs = [(DeviceDecoderState(st.req, st.buf, st.target_frames - min(lefts[i % len(lefts)], st.target_frames),
                                 st.target_frames), enc) for i, (enc, st) in enumerate(encs)]
    ref = [r.mel.frames for r in eng.decoder_batch(pairs)]
    print(f"B={B}: reference finite {all(np.isfinite(f).all() for f in ref)}", flush=True)
    names = ("U", "AP", "Gp", "Q", "P", "xb2", "mel", "work", "xbm", "G", "H1")
    for name in names:
        eng.poison_scratch = {name: float("nan")}
        try:
            got = [r.mel.frames for r in eng.decoder_batch(pairs)]
            bufs = eng._last_bufs
            if name == "AP":   # which (item, chunk) partial blocks were never written?
                ap = bufs.AP.float().cpu().numpy()
                Ls = [p[0].req.seq_len for p in pairs]
                missing = {b: [c for c in range(-(-L // 32)) if np.isnan(ap[b, c, 0])] for b, L in enumerate(Ls)}
                missing = {b: m for b, m in missing.items() if m}
                print(f"  AP never written (chunk 32 blocks): {len(missing)} items, e.g. "
                      f"{dict(list(missing.items())[:6])}; L of those {[Ls[b] for b in list(missing)[:6]]}", flush=True)
            if name in ("Gp", "Q", "P"):
                t = getattr(bufs, name).float().cpu().numpy()
                print(f"  {name}: NaN fraction after the call {np.isnan(t).mean():.3f}", flush=True)
            eng._last_bufs = None
        finally:
            eng.poison_scratch = {k: 0.0 for k in names}   # clean the allocator blocks again
            eng.decoder_batch(pairs)
            eng.poison_scratch = False
        bad = [i for i, (a, b) in enumerate(zip(ref, got)) if not np.array_equal(a, b)]
        nan = [i for i, g in enumerate(got) if not np.isfinite(g).all()]
        if bad:
            first = {i: int(np.argmax(np.any(ref[i] != got[i], axis=1))) for i in bad[:6]}
            print(f"  poison {name}: {len(bad)} items differ {bad[:12]} (non-finite {nan[:12]}); "
                  f"first differing frame {first}; steps {[ref[i].shape[0] for i in bad[:12]]}", flush=True)
        else:
            print(f"  poison {name}: no change", flush=True)
