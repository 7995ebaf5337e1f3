"""Non-incremental twin (baseline.py) vs the reference round semantics.

The reference ``run_round`` (``pkg/src/incrtts/baseline.py:61-141``) decodes every request to its
stop frame and delivers ``generate(whole mel)`` as ONE chunk at offset 0.  With the oracle Tier-S
modules behind the twin, each delivered waveform must equal the oracle's ``generate`` of the
concatenated mel exactly (fp64); with the GPU Tier-S modules within 1e-12 (the decoder frames
agree to ~1 ulp); and the RoundReport must carry the reference's fields.
"""

import numpy as np
import pytest

from oracle import tier_s as orc
from oracle.modules import cpu_modules
from paper_2211_13939_b200.baseline import BaselineServer, BaselineRequest, run_round
from paper_2211_13939_b200.frontend import run_frontend
from paper_2211_13939_b200.scheduler import ChunkStream, CostModel


def expected_waveform(text, lexicon, cfg):
    fo = run_frontend(text, lexicon)
    rows = orc.encode_rows(fo.phonemes, fo.pw, fo.pph, fo.iph, cfg.feature_dim)
    st = orc.init_state(rows.shape[0], cfg.feature_dim, cfg.frames_per_phoneme)
    mels = []
    while True:
        mel, stop, st = orc.decode_chunk(st, rows, cfg.chunk_frames, cfg.attention_penalty, cfg.stop_threshold)
        mels.append(mel)
        if stop:
            break
    return orc.generate(np.concatenate(mels, 0), cfg.hop_samples)


def check_round(modules, lexicon, cfg, texts, exact=True, tol=0.0):
    reqs = [BaselineRequest(i + 1, t, 0.0, ChunkStream(i + 1)) for i, t in enumerate(texts)]
    rep = run_round(reqs, modules, CostModel.zero(), cfg, round_index=3)
    assert rep.round_index == 3 and rep.request_ids == tuple(range(1, len(texts) + 1))
    assert rep.decoder_steps == max(rep.target_frames)
    for r, t in zip(reqs, texts):
        chunks = list(r.chunk_sink)
        assert len(chunks) == 1 and chunks[0].sample_offset == 0
        want = expected_waveform(t, lexicon, cfg)
        if exact:
            assert chunks[0].sample_count == want.shape[0]
            assert np.abs(chunks[0].samples - want).max() <= tol
        else:
            yield chunks[0].samples


def test_round_matches_reference_semantics_cpu(lexicon, cfg, texts):
    sample = [texts["short"][0], texts["medium"][0], texts["short"][1]]
    list(check_round(cpu_modules(lexicon, cfg), lexicon, cfg, sample))


def test_baseline_server_delivers_one_chunk_per_request(lexicon, cfg, texts):
    with BaselineServer(cpu_modules(lexicon, cfg), CostModel.zero(), cfg, max_batch=4) as srv:
        streams = [srv.submit(t)[1] for t in (texts["short"][0], texts["short"][1])]
        outs = [list(s) for s in streams]
    assert all(len(o) == 1 and o[0].sample_offset == 0 for o in outs)


@pytest.mark.gpu
def test_round_on_gpu_tier_s_bit_exact(lexicon, cfg, texts):
    from paper_2211_13939_b200.modules import build_modules
    mods = build_modules(lexicon, cfg, tier="s", device="cuda:0")
    sample = [texts["short"][0], texts["medium"][0], texts["long"][0]]
    # GPU decoder frames agree with the reference to ~1 ulp (dot-product order), see DESIGN.md
    list(check_round(mods, lexicon, cfg, sample, tol=1e-12))


@pytest.mark.gpu
def test_round_on_gpu_tier_r_whole_utterance(lexicon, cfg, texts):
    """Tier R: one whole-utterance waveform per request, length F*H, finite, non-silent."""
    from paper_2211_13939_b200.modules import build_modules
    mods = build_modules(lexicon, cfg, tier="r", device="cuda:0")
    sample = [texts["short"][0], texts["medium"][0]]
    reqs = [BaselineRequest(i + 1, t, 0.0, ChunkStream(i + 1)) for i, t in enumerate(sample)]
    rep = run_round(reqs, mods, CostModel.zero(), cfg)
    for r, target in zip(reqs, rep.target_frames):
        (chunk,) = list(r.chunk_sink)
        assert chunk.sample_offset == 0 and chunk.sample_count == target * cfg.hop_samples
        assert np.isfinite(chunk.samples).all() and np.abs(chunk.samples).max() > 0
