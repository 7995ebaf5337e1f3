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


@pytest.mark.parametrize("B", [1, 16, 100, 192, 256, 300, 512])
def test_persistent_matches_chain(engine, B):
    """Same (bf16) gate arithmetic on both paths; the split-bf16 parity mode is persistent-only."""
    engine.set_precision("bf16")
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
    engine.set_precision("parity")
    for a, b in zip(outs[True][0], outs[False][0]):
        assert np.isfinite(a).all()
        assert np.abs(a - b).max() <= 2e-4
    for sa, sb in zip(outs[True][1], outs[False][1]):
        for key in ("attn_weights", "attn_weights_sum", "attn_context", "dec_hidden", "dec_cell"):
            assert np.abs(sa[key] - sb[key]).max() <= 2e-4, key


def _ragged_pairs(engine, B, seed, lefts):
    """B fresh requests whose next chunk has `lefts[i % len]` frames left (mid-chunk stops)."""
    from paper_2211_13939_b200.handles import DeviceDecoderState
    lex = default_lexicon()
    encs = engine.encoder_batch([run_frontend(t, lex) for t in texts(B, seed)])
    pairs = []
    for i, (enc, st) in enumerate(encs):
        left = min(lefts[i % len(lefts)], st.target_frames)
        pairs.append((DeviceDecoderState(st.req, st.buf, st.target_frames - left, st.target_frames), enc))
    return pairs


@pytest.mark.parametrize("B", [3, 84, 120, 140, 300])
def test_scratch_is_written_before_read(engine, B):
    """NaN-filled decoder scratch (partials, attention numerators, operand mirror, outputs) must
    not change a single bit of the result: every scratch element the kernel reads was written
    earlier in the same launch.  Ragged stops (8 / 16 / 32 frames left) exercise the inactive-item
    paths of both the merged (B <= 96) and the separate chunk-combine schedule."""
    pairs = _ragged_pairs(engine, B, 100 + B, [8, 40, 64, 64, 16, 64, 48])
    got = {}
    for poison in (False, True):
        engine.poison_scratch = poison
        try:
            r1 = engine.decoder_batch(pairs)
            r2 = engine.decoder_batch([(r.state, enc) for r, (_, enc) in zip(r1, pairs) if not r.stop])
            got[poison] = ([r.mel.frames for r in r1] + [r.mel.frames for r in r2],
                           [engine.read_state(r.state.req, r.state.buf)["attn_weights_sum"] for r in r2])
        finally:
            engine.poison_scratch = False
    for a, b in zip(got[False][0], got[True][0]):
        assert np.isfinite(a).all() and np.array_equal(a, b)
    for a, b in zip(got[False][1], got[True][1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("B", [5, 84, 120, 300])
def test_graph_bucket_equals_eager(engine, B):
    """The CUDA-graph bucket (B padded to 16 with idle rows) gives the eager launch's bits."""
    pairs = _ragged_pairs(engine, B, 200 + B, [64, 64, 8, 40, 16])
    out = {}
    for graphs in (False, True):
        engine.use_graphs = graphs
        try:
            out[graphs] = [r.mel.frames for r in engine.decoder_batch(pairs)]
        finally:
            engine.use_graphs = False
    for a, b in zip(out[False], out[True]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("B", [24, 96, 97, 100, 136, 260, 512, 600])
def test_pooled_decode_equals_solo_bitwise(engine, B):
    """Batch transparency (reference SPEC.md:232, acceptance 1): a request's mel and state are the
    same bits whether it decodes alone or inside a pooled ragged batch (merged-combine B <= 96 and
    separate-combine schedules, one or two 256-row MMA N tiles, pools above 512 rows decoded in
    slices), over two consecutive chunks."""
    pairs = _ragged_pairs(engine, B, 300 + B, [64, 40, 8, 64, 16, 64])
    r1 = engine.decoder_batch(pairs)
    r2 = engine.decoder_batch([(r.state, enc) for r, (_, enc) in zip(r1, pairs) if not r.stop])
    pooled = [r.mel.frames for r in r1] + [r.mel.frames for r in r2]
    for i in sorted({0, 1, 2, B // 2, B - 1}):
        s1 = engine.decoder_batch([pairs[i]])[0]
        solo = [s1.mel.frames]
        if not s1.stop:
            solo.append(engine.decoder_batch([(s1.state, pairs[i][1])])[0].mel.frames)
        assert np.array_equal(solo[0], pooled[i])
        if len(solo) > 1:
            k = [j for j, r in enumerate(r1) if not r.stop].index(i)
            assert np.array_equal(solo[1], pooled[len(r1) + k])
