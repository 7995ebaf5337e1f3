"""Tier-S parity on the B200: CUDA kernels (through the C ABI) vs the reference.

Bit-exact: encoder rows, vocoder samples for given mel, chunk offsets and
counts, every IterationReport.  <= 1e-12: decoder frames / audio (the
reference's BLAS dot products are not order-pinned).  Mirrors the
reference's acceptance criteria 1, 2, 5, 10 (``pkg/tests/test_acceptance.py``).
"""

import math
import random

import numpy as np
import pytest

from oracle import tier_s as orc
from oracle.modules import cpu_modules
from paper_2211_13939_b200.domain import MelChunk, PipelineConfig
from paper_2211_13939_b200.frontend import FrontendOutput, run_frontend
from paper_2211_13939_b200.audio import VocoderState
from paper_2211_13939_b200.scheduler import CostModel, PipelineModules, RequestFailed, RequestPool, run_iteration

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engines():
    from paper_2211_13939_b200.modules import build_engine
    return {ol: build_engine(PipelineConfig(overlap_frames=ol), "s", "cuda:0") for ol in (4, 8)}


@pytest.fixture(scope="module")
def gpu_mods(engines, lexicon):
    from paper_2211_13939_b200.modules import modules_for
    return {ol: modules_for(e, lexicon) for ol, e in engines.items()}


def fo_from(arr):
    ph, pw, pph, iph = (tuple(int(x) for x in r) for r in arr)
    return FrontendOutput(ph, (len(ph),) + (0,) * (len(ph) - 1), pw, pph, iph)


def table(reports):
    return [[list(r.frontend_ids), list(r.encoder_ids), list(r.decoder_ids), list(r.vocoder_ids),
             list(r.completed_ids), list(r.failed_ids)] for r in reports]


def drain(pool, mods, cfg):
    reps = []
    while pool.pending():
        reps.append(run_iteration(pool, mods, CostModel.zero(), cfg, step_index=len(reps)))
    return reps


def random_texts(lexicon, count, seed, lo=2, hi=12):
    singles = sorted(c for c in lexicon.phrase_to_pinyin if len(c) == 1)
    rng = random.Random(seed)
    return ["".join(rng.choice(singles) for _ in range(rng.randint(lo, hi))) for _ in range(count)]


def test_encoder_rows_bit_exact(engines, golden_units):
    fos = [fo_from(golden_units[f"enc_in_{i}"]) for i in range(25)]
    out = engines[4].encoder_batch(fos)
    for i, (enc, state) in enumerate(out):
        assert np.array_equal(enc.rows, golden_units[f"enc_rows_{i}"]), i
        assert state.frames_emitted == 0 and state.target_frames == 8 * fos[i].seq_len
        assert np.array_equal(state.attn_weights_sum, np.zeros(fos[i].seq_len))


def test_decoder_trace_matches_reference(engines, golden_units):
    eng = engines[4]
    for i in range(3):
        (enc, st), = eng.encoder_batch([fo_from(golden_units[f"dec_in_{i}"])])
        want = golden_units[f"dec_frames_{i}"]
        got, k = [], 0
        while k < want.shape[0] and st.frames_emitted < st.target_frames:
            res, = eng.decoder_batch([(st, enc)])
            got.append(res.mel.frames)
            k += res.mel.frame_count
            st = res.state
        got = np.concatenate(got)[:want.shape[0]]
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


def test_batched_decode_equals_sequential_and_values_persist(engines, golden_units):
    eng = engines[4]
    fos = [fo_from(golden_units[f"enc_in_{i}"]) for i in range(10)]
    pairs = [(s, e) for e, s in eng.encoder_batch(fos)]
    batched = eng.decoder_batch(pairs)
    for (st, enc), res in zip(pairs, batched):  # old handles still valid: value semantics
        solo, = eng.decoder_batch([(st, enc)])
        assert np.array_equal(res.mel.frames, solo.mel.frames)
        assert res.stop == solo.stop and res.state.frames_emitted == solo.state.frames_emitted
        assert np.array_equal(res.state.attn_weights_sum, solo.state.attn_weights_sum)


def test_decode_errors(engines):
    eng = engines[4]
    (e1, s1), (e2, s2) = eng.encoder_batch([fo_from([[1], [0], [0], [1]]), fo_from([[1, 2], [0, 0], [0, 0], [0, 1]])])
    with pytest.raises(ValueError, match="does not match"):
        eng.decoder_batch([(s1, e2)])
    res, = eng.decoder_batch([(s1, e1)])
    assert res.stop and res.mel.frame_count == 8
    with pytest.raises(ValueError, match="past stop"):
        eng.decoder_batch([(res.state, e1)])


@pytest.mark.parametrize("ol", [4, 8])
def test_vocoder_splices_bit_exact(engines, golden_units, ol):
    eng = engines[ol]
    for j in range(5):
        key = f"voc_ol{ol}_{j}"
        mel, lens = golden_units[key + "_mel"], golden_units[key + "_lens"]
        st, start, got, offs = VocoderState.initial(), 0, [], []
        for k, m in enumerate(lens):
            (audio, st), = eng.vocoder_batch([(st, MelChunk(mel[start:start + m]), k == len(lens) - 1)])
            got.append(audio.samples), offs.append(audio.sample_offset)
            start += m
        assert offs == list(golden_units[key + "_offsets"])
        assert np.array_equal(np.concatenate(got), golden_units[key + "_samples"])


def test_vocoder_rejects_short_non_final(engines):
    with pytest.raises(ValueError, match="overlap"):
        engines[4].vocoder_batch([(VocoderState.initial(), MelChunk(np.zeros((3, 8))), False)])


@pytest.mark.parametrize("ol", [4, 8])
def test_pipeline_matches_reference_synthesis(gpu_mods, golden_synth, golden_frontend, ol):
    cfg = PipelineConfig(overlap_frames=ol)
    pool = RequestPool()
    streams = [pool.submit(t)[1] for t in golden_frontend["texts"]]
    drain(pool, gpu_mods[ol], cfg)
    for i, stream in enumerate(streams):
        chunks = list(stream)
        key = f"ol{ol}_{i}"
        assert [c.sample_offset for c in chunks] == list(golden_synth[key + "_offsets"])
        assert [c.sample_count for c in chunks] == list(golden_synth[key + "_counts"])
        np.testing.assert_allclose(np.concatenate([c.samples for c in chunks]),
                                   golden_synth[key + "_samples"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("ol", [4, 8])
def test_fig2_and_random_schedules(gpu_mods, golden_schedules, ol):
    cfg = PipelineConfig(overlap_frames=ol)
    mods = gpu_mods[ol]
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
    assert table(reps) == golden_schedules[f"fig2_ol{ol}"]
    name = "random_a" if ol == 4 else "random_b"
    pool, reps = RequestPool(), []
    for batch in golden_schedules[name]["script"]:
        for text in batch:
            pool.submit(text)
        step()
    assert table(reps) == golden_schedules[name]["table"]


def test_acceptance_01_batch_transparency(gpu_mods, lexicon, cfg):
    texts = random_texts(lexicon, 100, seed=101)
    pool = RequestPool()
    streams = [pool.submit(t)[1] for t in texts]
    drain(pool, gpu_mods[4], cfg)
    for text, stream in zip(texts, streams):
        fo = run_frontend(text, lexicon)
        want, _ = orc.synthesize(fo.phonemes, fo.pw, fo.pph, fo.iph)
        got = list(stream)
        assert [c.sample_offset for c in got] == [o for _, o in want]
        for g, (w, _) in zip(got, want):
            assert g.samples.shape == w.shape
            assert np.max(np.abs(g.samples - w)) <= 1e-12


@pytest.mark.parametrize("ol", [4, 8])
def test_acceptance_05_10_stream_conservation(gpu_mods, lexicon, ol):
    cfg = PipelineConfig(overlap_frames=ol)
    pool_texts = random_texts(lexicon, 60, seed=505 + ol)
    rng = random.Random(ol)
    texts = [rng.choice(pool_texts) for _ in range(1000)]
    pool = RequestPool()
    streams = [(t, pool.submit(t)[1]) for t in texts]
    drain(pool, gpu_mods[ol], cfg)
    for text, stream in streams:
        target = cfg.frames_per_phoneme * run_frontend(text, lexicon).seq_len
        offset, chunks = 0, list(stream)
        for c in chunks:
            assert c.sample_offset == offset
            offset += c.sample_count
        assert offset == target * cfg.hop_samples
        assert len(chunks) == math.ceil(target / cfg.chunk_frames)


def test_long_paragraph_matches_oracle(gpu_mods, lexicon, cfg):
    text = random_texts(lexicon, 1, seed=77, lo=300, hi=300)[0]
    short = random_texts(lexicon, 5, seed=78, lo=2, hi=20)
    pool = RequestPool()
    streams = [pool.submit(t)[1] for t in [text] + short]
    drain(pool, gpu_mods[4], cfg)
    for t, stream in zip([text] + short, streams):
        fo = run_frontend(t, lexicon)
        want, _ = orc.synthesize(fo.phonemes, fo.pw, fo.pph, fo.iph)
        got = np.concatenate([c.samples for c in stream])
        np.testing.assert_allclose(got, np.concatenate([w for w, _ in want]), rtol=0, atol=1e-12)


def test_decoder_fault_isolated(gpu_mods, cfg):
    mods = gpu_mods[4]
    target = {"id": None}

    def decoder(pairs):
        out = []
        for st, enc in pairs:
            if target["id"] is not None and st.frames_emitted >= 64:
                raise RuntimeError("decoder fault")
            out.extend(mods.decoder_batch([(st, enc)]))
        return out

    faulty = PipelineModules(mods.frontend_batch, mods.encoder_batch, decoder, mods.vocoder_batch)
    pool = RequestPool()
    long_id, long_stream = pool.submit("欢迎大家收听今天下午新闻播报")
    _, short_stream = pool.submit("你们好")
    target["id"] = long_id
    drain(pool, faulty, cfg)
    got = []
    with pytest.raises(RequestFailed):
        for c in long_stream:
            got.append(c)
    assert len(got) == 2 and len(list(short_stream)) == 2


def test_arena_is_released(engines, lexicon, cfg):
    import gc
    from paper_2211_13939_b200.modules import modules_for
    eng = engines[4]
    gc.collect()
    before = eng.arena.used
    pool = RequestPool()
    for t in random_texts(lexicon, 50, seed=9):
        pool.submit(t)
    drain(pool, modules_for(eng, lexicon), cfg)
    gc.collect()
    assert eng.arena.used == before
