import sys, random
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2211_13939_b200.domain import PipelineConfig
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend
from paper_2211_13939_b200.harness import random_text
from paper_2211_13939_b200.tier_r import TierREngine
eng = TierREngine(PipelineConfig(), "cuda:0")
lex = default_lexicon()
rng = random.Random(21)
for B in (5, 16, 24):
    fos = [run_frontend(random_text(rng, 8, 30, lex), lex) for _ in range(B)]
    pairs = [(st, enc) for enc, st in eng.encoder_batch(fos)]
    outs = {}
    for mode in ("eager", "eager2", "graph", "graph2"):
        eng.use_graphs = mode.startswith("graph")
        outs[mode] = eng.decoder_batch(pairs)
    for m in ("eager2", "graph", "graph2"):
        d = max(float(np.abs(a.mel.frames - b.mel.frames).max()) for a, b in zip(outs["eager"], outs[m]))
        dw = max(float(np.abs(a.state.attn_weights_sum - b.state.attn_weights_sum).max()) for a, b in zip(outs["eager"], outs[m]))
        print(B, m, "mel maxdiff", d, "attn_sum maxdiff", dw)
