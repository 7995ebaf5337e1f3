"""Reproduce the round-based twin's decoder calls (3 items: short / medium / long fixture texts)
and report which decoder call first produces non-finite mel, per precision / graph setting."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, default_texts, run_frontend  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

eng = TierREngine(PipelineConfig(), "cuda:0")
lex, texts = default_lexicon(), default_texts()
sample = [texts["short"][0], texts["medium"][0], texts["long"][0]]
for prec in ("parity", "bf16"):
    for graphs in (True, False):
        for rep in range(3):
            eng.set_precision(prec)
            eng.use_graphs = graphs
            encs = eng.encoder_batch([run_frontend(t, lex) for t in sample])
            states = {i: (st, enc) for i, (enc, st) in enumerate(encs)}
            call, bad = 0, []
            while states:
                order = sorted(states)
                res = eng.decoder_batch([states[i] for i in order])
                for i, r in zip(order, res):
                    f = r.mel.frames
                    if not np.isfinite(f).all():
                        bad.append((call, i, len(order), r.mel.frame_count, int(np.argmax(~np.isfinite(f).all(1)))))
                    if r.stop:
                        del states[i]
                    else:
                        states[i] = (r.state, states[i][1])
                call += 1
            print(f"{prec} graphs={graphs} rep {rep}: {call} calls, non-finite (call, item, batch, frames, first bad frame): {bad}", flush=True)
