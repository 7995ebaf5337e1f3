"""Persistent decoder kernel (dec_persist.cu) vs the per-kernel decoder chain on the same inputs.

Both paths compute the same Tacotron2 decoder steps in the same precision (bf16 gate GEMMs with
fp32 accumulation, fp32 elsewhere) but with different reduction orders, so a chunk of 32 steps
must agree to well inside the oracle tolerance (mel max-abs 1e-3): 2e-4 here.  Batch sizes cover
one and two 128-item blocks of the operand mirror and ragged text lengths.
"""

import random

import numpy as np
import pytest
import torch

from paper_2211_13939_b200.domain import PipelineConfig
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2211_13939_b200.tier_r import TierREngine
    eng = TierREngine(PipelineConfig(), "cuda:0")
    eng.use_graphs = False
    return eng


def texts(n, seed, lo=20, hi=200):
    lex = default_lexicon()
    singles = sorted(c for c in lex.phrase_to_pinyin if len(c) == 1)
    rng = random.Random(seed)
    return ["".join(rng.choice(singles) for _ in range(rng.randint(lo, hi))) for _ in range(n)]


@pytest.mark.parametrize("B", [1, 16, 100, 192, 256])
def test_persistent_matches_chain(engine, B):
    lex = default_lexicon()
    encs = engine.encoder_batch([run_frontend(t, lex) for t in texts(B, B)])
    pairs = [(st, enc) for enc, st in encs]
    # two chunks: the second starts from a state the first produced (W / W_acc / cells / h)
    outs = {}
    for persistent in (True, False):
        engine.persistent_decoder = persistent
        r1 = engine.decoder_batch(pairs)
        r2 = engine.decoder_batch([(r.state, enc) for r, (_, enc) in zip(r1, pairs)])
        torch.cuda.synchronize()
        outs[persistent] = ([r.mel.frames for r in r1] + [r.mel.frames for r in r2],
                            [engine.read_state(r.state.req, r.state.buf) for r in r2])
    engine.persistent_decoder = True
    for a, b in zip(outs[True][0], outs[False][0]):
        assert np.isfinite(a).all()
        assert np.abs(a - b).max() <= 2e-4
    for sa, sb in zip(outs[True][1], outs[False][1]):
        for key in ("attn_weights", "attn_weights_sum", "attn_context", "dec_hidden", "dec_cell"):
            assert np.abs(sa[key] - sb[key]).max() <= 2e-4, key
