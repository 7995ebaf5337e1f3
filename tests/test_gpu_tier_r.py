"""Tier-R parity on the B200: Tacotron2 + HiFi-GAN V1 CUDA path vs the torch-CPU fp32 oracle.

Tolerances (stated in north_star): mel max-abs <= 1e-3, waveform SNR >= 40 dB,
chunk offsets / counts / stop steps / IterationReports exact.  The oracle
is the builder's restatement (the reference has no networks), so these
pins are "parity unpinned by the reference" -- see DESIGN.md.
"""

import math
import random

import numpy as np
import pytest
import torch

from oracle import tier_r as orc
from oracle import tier_s as orc_s
from paper_2211_13939_b200.audio import VocoderState
from paper_2211_13939_b200.domain import MelChunk, PipelineConfig
from paper_2211_13939_b200.frontend import run_frontend
from paper_2211_13939_b200.scheduler import CostModel, RequestPool, run_iteration
from paper_2211_13939_b200.weights import tier_r_weights

pytestmark = pytest.mark.gpu
MEL_TOL = 1e-3
SNR_DB = 40.0


@pytest.fixture(scope="module")
def weights():
    return tier_r_weights(0)


@pytest.fixture(scope="module")
def engine(weights):
    from paper_2211_13939_b200.tier_r import TierREngine
    return TierREngine(PipelineConfig(), "cuda:0", weights=weights)


def random_texts(lexicon, count, seed, lo, hi):
    singles = sorted(c for c in lexicon.phrase_to_pinyin if len(c) == 1)
    rng = random.Random(seed)
    return ["".join(rng.choice(singles) for _ in range(rng.randint(lo, hi))) for _ in range(count)]


def run_direct(engine, fos, max_chunks=None):
    """Module calls in batch (all items together), like run_iteration without admission."""
    encs = engine.encoder_batch(fos)
    live = [(i, enc, st, VocoderState.initial()) for i, (enc, st) in enumerate(encs)]
    mels = [[] for _ in fos]
    audio = [[] for _ in fos]
    rounds = 0
    while live:
        res = engine.decoder_batch([(st, enc) for _, enc, st, _ in live])
        outs = engine.vocoder_batch([(vs, r.mel, r.stop) for (_, _, _, vs), r in zip(live, res)])
        nxt = []
        for (i, enc, _, _), r, (a, vs) in zip(live, res, outs):
            mels[i].append(r.mel.frames)
            audio[i].append((a.samples.copy(), a.sample_offset))
            if not r.stop:
                nxt.append((i, enc, r.state, vs))
        live = nxt
        rounds += 1
        if max_chunks and rounds >= max_chunks:
            break
    return mels, audio


def test_encoder_matches_oracle(engine, weights, lexicon):
    texts = ["欢迎收听今天新闻。", "你们好"] + random_texts(lexicon, 3, 5, 20, 60)
    fos = [run_frontend(t, lexicon) for t in texts]
    encs = engine.encoder_batch(fos)
    for fo, (enc, st) in zip(fos, encs):
        mem, pm = orc.encode(weights, fo.phonemes, fo.pw, fo.pph, fo.iph)
        got = enc.rows
        assert got.shape == tuple(mem.shape)
        # default split-bf16 parity mode: fp32-level products (measured ~6e-6 / 1e-5); bf16 mode ~1e-3
        assert np.abs(got - mem.numpy()).max() <= 5e-5, np.abs(got - mem.numpy()).max()
        gpm = engine.read_processed_memory(enc.req)
        assert np.abs(gpm - pm.numpy()).max() <= 5e-5
        assert st.frames_emitted == 0 and st.target_frames == 8 * fo.seq_len


def test_pre_encoded_requests_decode_identically(engine, lexicon):
    """pre_encode (frontend outputs prefetched during a vocoder wait, encoded right then): the
    admitting encoder_batch returns those results, and decoding / vocoding them gives the same
    bits as encoding at admission."""
    fos = [run_frontend(t, lexicon) for t in random_texts(lexicon, 5, 321, 10, 60)]
    outs = []
    for pre in (False, True):
        if pre:
            engine.pre_encode(fos[1:4])
        hits = engine.pre_enc_hits
        encs = engine.encoder_batch(fos)
        assert engine.pre_enc_hits - hits == (3 if pre else 0)
        res = engine.decoder_batch([(st, enc) for enc, st in encs])
        audio = engine.vocoder_batch([(VocoderState.initial(), r.mel, r.stop) for r in res])
        outs.append([(np.asarray(r.mel.frames), a.samples.copy()) for r, (a, _) in zip(res, audio)])
    for (m0, a0), (m1, a1) in zip(*outs):
        assert np.array_equal(m0, m1) and np.array_equal(a0, a1)


def test_tensor_core_bilstm_matches_oracle(weights, lexicon, monkeypatch):
    """Opt-in tensor-core BiLSTM (ITTS_BILSTM_TC=1, pooled encoder batches >= 96 items): encoder
    memory within the same fp32-level tolerance of the oracle as the SIMT recurrence."""
    from paper_2211_13939_b200.tier_r import TierREngine
    monkeypatch.setenv("ITTS_BILSTM_TC", "1")
    eng = TierREngine(PipelineConfig(), "cuda:0", weights=weights)
    assert eng.enc_whh_tc is not None
    texts = random_texts(lexicon, 100, 77, 5, 40)
    fos = [run_frontend(t, lexicon) for t in texts]
    encs = eng.encoder_batch(fos)
    for i in (0, 37, 99):
        mem, _ = orc.encode(weights, fos[i].phonemes, fos[i].pw, fos[i].pph, fos[i].iph)
        err = np.abs(encs[i][0].rows - mem.numpy()).max()
        assert err <= 5e-5, (i, err)


@pytest.mark.parametrize("n", [12, 40, 128])
def test_pooled_encoder_is_bitwise_transparent(engine, lexicon, n):
    """Each item's encoder memory in a pooled ragged batch (packed rows, shared convs, one BiLSTM
    cluster per item) is the same bits as when it is encoded alone (batch transparency,
    SPEC.md:232)."""
    fos = [run_frontend(t, lexicon) for t in random_texts(lexicon, n, 100 + n, 20, 200)]
    encs = engine.encoder_batch(fos)
    pooled = {i: encs[i][0].rows.copy() for i in sorted({0, 1, n // 2, n - 1})}
    for i, rows in pooled.items():
        (enc, _), = engine.encoder_batch([fos[i]])
        assert np.array_equal(enc.rows, rows), i


def test_vocoder_chunks_match_oracle(engine, weights):
    rng = np.random.default_rng(3)
    for lens, last_short in (((32, 32, 8), False), ((16,), False), ((32, 2), True)):
        mels = [rng.uniform(-0.1, 0.1, size=(m, 80)) for m in lens]
        st_g, st_o = VocoderState.initial(), orc_s.VocState(None, None, 0)
        for k, m in enumerate(mels):
            last = k == len(mels) - 1
            (a, st_g), = engine.vocoder_batch([(st_g, MelChunk(m), last)])
            want, off, st_o = orc.vocode_chunk(weights, st_o, m, last, 4)
            assert a.sample_offset == off and a.sample_count == want.size
            assert orc.snr_db(want, a.samples) >= SNR_DB, orc.snr_db(want, a.samples)


def test_batched_vocoder_equals_solo(engine):
    rng = np.random.default_rng(4)
    triples = [(VocoderState.initial(), MelChunk(rng.uniform(-0.1, 0.1, (m, 80))), last)
               for m, last in ((32, False), (20, True), (32, False), (7, True))]
    batched = engine.vocoder_batch(triples)
    for t, (a, _) in zip(triples, batched):
        (solo, _), = engine.vocoder_batch([t])
        assert np.array_equal(a.samples, solo.samples)  # batch invariance: same kernels, same order


def test_end_to_end_mel_and_audio(engine, weights, lexicon):
    texts = ["欢迎收听今天新闻。", "你们好", "欢迎大家收听今天下午新闻播报"]
    fos = [run_frontend(t, lexicon) for t in texts]
    mels, audio = run_direct(engine, fos)
    for fo, m, au in zip(fos, mels, audio):
        chunks, mel_ref, _ = orc.synthesize(weights, fo.phonemes, fo.pw, fo.pph, fo.iph)
        got = np.concatenate(m)
        assert got.shape == mel_ref.shape
        err = np.abs(got - mel_ref).max()
        print(f"mel max-abs err {err:.3e} over {got.shape[0]} frames")
        assert err <= MEL_TOL, err
        assert [o for _, o in au] == [o for _, o in chunks]
        assert [s.size for s, _ in au] == [s.size for s, _ in chunks]
        snr = orc.snr_db(np.concatenate([s for s, _ in chunks]), np.concatenate([s for s, _ in au]))
        print(f"waveform SNR {snr:.1f} dB")
        assert snr >= SNR_DB, snr


def test_schedule_identical_to_reference(engine, golden_schedules, lexicon):
    from paper_2211_13939_b200.modules import modules_for
    mods = modules_for(engine, lexicon)
    cfg = PipelineConfig()
    pool, reps = RequestPool(), []
    step = lambda: reps.append(run_iteration(pool, mods, CostModel.zero(), cfg, step_index=len(reps)))
    four, five = "欢迎收听新闻播报", "欢迎收听今天新闻。"
    pool.submit(four); step(); step()
    pool.submit(four); pool.submit(five)
    for _ in range(4):
        step()
    pool.submit(four); step()
    while pool.pending():
        step()
    table = [[list(r.frontend_ids), list(r.encoder_ids), list(r.decoder_ids), list(r.vocoder_ids),
              list(r.completed_ids), list(r.failed_ids)] for r in reps]
    assert table == golden_schedules["fig2_ol4"]


def test_stream_conservation_ragged_pool(engine, lexicon):
    from paper_2211_13939_b200.modules import modules_for
    mods = modules_for(engine, lexicon)
    cfg = PipelineConfig()
    texts = random_texts(lexicon, 40, 11, 1, 40)
    pool = RequestPool()
    streams = [(t, pool.submit(t)[1]) for t in texts]
    while pool.pending():
        run_iteration(pool, mods, CostModel.zero(), cfg)
    for text, stream in streams:
        target = 8 * run_frontend(text, lexicon).seq_len
        chunks, off = list(stream), 0
        for c in chunks:
            assert c.sample_offset == off
            off += c.sample_count
        assert off == target * 256 and len(chunks) == math.ceil(target / 32)


def test_graph_replay_equals_eager(engine, lexicon):
    """CUDA-graph bucket path and eager launches give bit-identical chunks (fixed reduction orders)."""
    texts = random_texts(lexicon, 5, 21, 8, 30)
    fos = [run_frontend(t, lexicon) for t in texts]
    pairs = [(st, enc) for enc, st in engine.encoder_batch(fos)]
    engine.use_graphs = False
    try:
        eager = engine.decoder_batch(pairs)
    finally:
        engine.use_graphs = True
    graph = engine.decoder_batch(pairs)
    graph2 = engine.decoder_batch(pairs)  # replay of the captured graph
    for e, g, g2 in zip(eager, graph, graph2):
        assert np.array_equal(e.mel.frames, g.mel.frames)
        assert np.array_equal(g.mel.frames, g2.mel.frames)
        assert np.array_equal(e.state.attn_weights_sum, g.state.attn_weights_sum)
        assert np.array_equal(e.state.dec_hidden, g2.state.dec_hidden)


def test_device_pcm16_matches_reference_encoding(engine, lexicon):
    """f1: PCM16 produced in the splice pass == pcm16_encode of the float chunk, bit-exact."""
    from paper_2211_13939_b200.audio import pcm16_encode
    engine.pcm16 = True
    try:
        fos = [run_frontend(t, lexicon) for t in random_texts(lexicon, 3, 11, 20, 60)]
        encs = engine.encoder_batch(fos)
        live = [(enc, st, VocoderState.initial()) for enc, st in encs]
        checked = 0
        while live and checked < 6:
            res = engine.decoder_batch([(st, enc) for enc, st, _ in live])
            outs = engine.vocoder_batch([(vs, r.mel, r.stop) for (_, _, vs), r in zip(live, res)])
            for chunk, _ in outs:
                assert chunk.pcm16() == pcm16_encode(chunk.samples)
                assert "_pcm16" in chunk.__dict__
            checked += 1
            live = [(enc, r.state, vs) for (enc, _, _), r, (_, vs) in zip(live, res, outs) if not r.stop]
    finally:
        engine.pcm16 = False


def test_device_wire_base64_matches_reference_server(engine, lexicon):
    """f1 wire format: the base64 text of each chunk's PCM16, produced on device, equals the
    reference server's encode_samples (src/server.py:78-79) of the float chunk -- for ragged
    chunk lengths, including the final short chunks (all three '=' padding cases occur)."""
    import base64

    from paper_2211_13939_b200.audio import pcm16_encode
    engine.wire_b64 = True
    pads = set()
    try:
        fos = [run_frontend(t, lexicon) for t in random_texts(lexicon, 5, 12, 3, 40)]
        encs = engine.encoder_batch(fos)
        live = [(enc, st, VocoderState.initial()) for enc, st in encs]
        while live:
            res = engine.decoder_batch([(st, enc) for enc, st, _ in live])
            outs = engine.vocoder_batch([(vs, r.mel, r.stop) for (_, _, vs), r in zip(live, res)])
            for chunk, _ in outs:
                assert "_b64" in chunk.__dict__
                want = base64.b64encode(pcm16_encode(chunk.samples)).decode("ascii")
                assert chunk.wire_samples() == want
                pads.add((2 * chunk.sample_count) % 3)
            live = [(enc, r.state, vs) for (enc, _, _), r, (_, vs) in zip(live, res, outs) if not r.stop]
    finally:
        engine.wire_b64 = False
    assert len(pads) >= 2, pads


@pytest.mark.parametrize("sizes", [(1,), (5, 3, 40), (24,)])
def test_native_vocoder_sequence_equals_python_launches(engine, sizes):
    """voc_run.cu (C++ launch sequence, 1 or 3 streams) == the per-layer Python launch loop, bit-exact."""
    rng = np.random.default_rng(sum(sizes))
    triples = []
    for k, B in enumerate(sizes):
        for i in range(B):
            m = int(rng.integers(1, 33)) if i % 7 == 3 else 32
            triples.append((VocoderState.initial(), MelChunk(rng.uniform(-0.2, 0.2, (m, 80))), m < 32))
    got = {}
    for native in (False, True):
        for streams in (False, True):
            engine.native_vocoder, engine.mrf_streams = native, streams
            try:
                got[native, streams] = [a.samples for a, _ in engine.vocoder_batch(triples)]
            finally:
                engine.native_vocoder, engine.mrf_streams = True, True
    want = got[False, False]
    for key, outs in got.items():
        for a, b in zip(outs, want):
            assert np.array_equal(a, b), key


def test_native_vocoder_large_pool(engine):
    """A 256-chunk pooled call through voc_run (host frame table, grown work buffers) matches solo calls."""
    rng = np.random.default_rng(9)
    triples = [(VocoderState.initial(), MelChunk(rng.uniform(-0.2, 0.2, (32, 80))), False) for _ in range(256)]
    batched = engine.vocoder_batch(triples)
    for i in (0, 131, 255):
        (solo, _), = engine.vocoder_batch([triples[i]])
        assert np.array_equal(batched[i][0].samples, solo.samples)


def test_vocoder_ignores_unwritten_buffer_contents(engine, weights, monkeypatch):
    """Every row the HiFi-GAN sequence reads (halos included) is written inside the same call:
    work buffers filled with bf16 NaN at allocation (ITTS_VOC_POISON=1) give the same bits.
    (compute-sanitizer initcheck cannot show this: it does not track TMA tensor stores.)"""
    from paper_2211_13939_b200.tier_r import TierREngine
    rng = np.random.default_rng(21)
    triples = [(VocoderState.initial(), MelChunk(rng.uniform(-0.2, 0.2, (m, 80))), m < 32)
               for m in (32, 5, 32, 17, 32, 1, 32, 32)]
    want = [a.samples for a, _ in engine.vocoder_batch(triples)]
    monkeypatch.setenv("ITTS_VOC_POISON", "1")
    poisoned = TierREngine(PipelineConfig(), "cuda:0", weights=weights)
    for sub in (triples, triples[:3], triples):   # fresh buffers, then reuse after a smaller call
        got = [a.samples for a, _ in poisoned.vocoder_batch(sub)]
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


def test_nonfinite_audio_is_caught_on_device(engine):
    """The finite-audio guard (reference _frozen_array, domain.py:170-178) now counts non-finite
    samples per chunk in the splice kernel: an overflowing mel chunk fails its batch (the
    scheduler then isolates it per item) and a good chunk alone still passes."""
    good = (VocoderState.initial(), MelChunk(np.zeros((32, 80))), False)
    bad = (VocoderState.initial(), MelChunk(np.full((32, 80), 3e38)), False)
    with pytest.raises(ValueError, match="non-finite"):
        engine.vocoder_batch([good, bad])
    (chunk, _), = engine.vocoder_batch([good])
    assert np.isfinite(chunk.samples).all()


def test_chunks_stay_valid_while_held(engine):
    """Chunks are read-only views of pinned D2H slots; a slot is reused only once no chunk views
    it, so chunks held across many later calls keep their samples."""
    rng = np.random.default_rng(3)
    held = []
    for it in range(10):
        triples = [(VocoderState.initial(), MelChunk(rng.uniform(-0.3, 0.3, (32, 80))), False) for _ in range(3)]
        out = engine.vocoder_batch(triples)
        held += [(c, c.samples.copy()) for c, _ in out]
    for c, ref in held:
        assert np.array_equal(c.samples, ref)
        assert not c.samples.flags.writeable


def test_serving_replay_matches_serialized_launches():
    """A deterministic serving replay (arrivals, stops, pooled batches) gives bit-identical chunks
    with the default launch configuration (MRF branches on 3 streams, decoder speculation) and a
    fully serialised one (one stream, no speculation, no PDL): no cross-kernel / cross-stream race."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    outs = []
    for extra, env_add in (([], {}), (["--serial"], {"ITTS_NO_PDL": "1"})):
        env = dict(os.environ, **env_add)
        out = subprocess.run([sys.executable, str(root / "tools" / "race_check.py"), "--iters", "150", *extra],
                             env=env, cwd=root, capture_output=True, text=True, timeout=900)
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(out.stdout.strip().splitlines()[-1])
    assert outs[0].startswith("failed/non-finite 0;"), outs
    assert outs[0] == outs[1], outs


def test_decoder_launch_speculation_is_transparent():
    """Large pools launch the continuing items' next decoder chunk during the vocoder wait
    (engine.spec_launch_min); with the threshold lowered so every iteration speculates, the
    deterministic serving replay gives the same chunk digest as fully serialised launches."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    outs = []
    for extra in (["--spec-launch-min", "4"], ["--serial"]):
        env = dict(os.environ, ITTS_NO_PDL="1")
        out = subprocess.run([sys.executable, str(root / "tools" / "race_check.py"), "--iters", "120", "--heavy",
                              *extra], env=env, cwd=root, capture_output=True, text=True, timeout=900)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = out.stdout.strip().splitlines()
        outs.append(lines[-1])
        if extra[0] == "--spec-launch-min":
            hits = int(lines[-2].split()[-1])
            assert hits > 0, lines[-2]
    assert outs[0].startswith("failed/non-finite 0;"), outs
    assert outs[0] == outs[1], outs


def test_chunk_postnet_matches_oracle(engine, lexicon):
    """f3: mel + PostNet(mel) per chunk (tensor-core convs, bf16 activations) vs the fp32 oracle."""
    from paper_2211_13939_b200.weights import postnet_weights
    pw = postnet_weights(0)
    fos = [run_frontend(t, lexicon) for t in random_texts(lexicon, 5, 31, 8, 40)]
    pairs = [(st, enc) for enc, st in engine.encoder_batch(fos)]
    for graphs in (True, False):
        engine.use_graphs = graphs
        try:
            engine.set_postnet(False)
            pre = engine.decoder_batch(pairs)
            engine.set_postnet(True, pw)
            post = engine.decoder_batch(pairs)
        finally:
            engine.set_postnet(False)
            engine.use_graphs = True
        for a, b in zip(pre, post):
            assert a.mel.frame_count == b.mel.frame_count and a.stop == b.stop
            want = orc.postnet(pw, a.mel.frames)
            got = np.asarray(b.mel.frames)
            assert np.abs(got - want).max() <= 5e-2, np.abs(got - want).max()
            assert np.sqrt(np.mean((got - want) ** 2)) <= 1e-2 * max(1.0, np.sqrt(np.mean(want ** 2)))
            # the fed-back state is the pre-PostNet frame: both calls leave the same decoder state
            assert np.array_equal(a.state.dec_hidden, b.state.dec_hidden)
