"""Pins the Tier-S oracle to vectors produced by the reference itself.

Golden data: ``tests/golden/tier_s_units.npz`` / ``tier_s_synth.npz``
(``tools/make_golden.py``).  Frozen constants below are the reference
tests' own (``pkg/tests/test_domain.py:40-47``,
``pkg/tests/test_acoustic.py:32-47``).
"""

import numpy as np
import pytest

from oracle import tier_s

SEEDED_TABLE0_TOKEN5 = [
    -0.01400420279972603, 0.36631764218069907, -0.24983897799184018, -0.12769336388567454,
    -0.45611580533145535, 0.45329481155484275, 0.80959633298746181, 0.30866268294702826]
FIXTURE_ENCODER_ROWS = [
    [-0.12233080011854928, 0.29807743169234407, -0.85580035060658100, 1.40008302978261145,
     -2.53872254635790062, -0.36117914215327440, -1.00869400099871953, 0.48956677142731619],
    [0.81484723133181192, 0.14873783020264428, -1.28369211272811534, 0.92564941793718936,
     -1.54443796088616181, -0.93108128061454210, 0.31989735213923370, 1.21856747910382102],
    [0.91493732342417111, 0.18529284119704903, -0.17214746298859884, 0.89315055752199424,
     -1.41862066965575084, 0.13733758247793273, 0.27370803570560603, 1.15959640821779786]]
FIXTURE_STEP_FRAME = [
    0.65936100759619964, 0.30523488434817242, -0.80831732688679236, 0.90998389691319059,
    -0.98532190404171027, -0.51745653460105057, -0.20440420665301431, 0.87945658345739297]


def test_seeded_vectors_bit_exact(golden_units):
    toks = golden_units["seeded_tokens"]
    for table in range(4):
        got = tier_s.seeded_vectors(table, toks, 16)
        assert np.array_equal(got, golden_units[f"seeded_t{table}"])
    np.testing.assert_allclose(tier_s.seeded_vector(0, 5, 8), SEEDED_TABLE0_TOKEN5, rtol=0, atol=1e-12)


def test_encoder_rows_bit_exact(golden_units):
    for i in range(25):
        ph, pw, pph, iph = golden_units[f"enc_in_{i}"]
        assert np.array_equal(tier_s.encode_rows(ph, pw, pph, iph, 8), golden_units[f"enc_rows_{i}"])


def test_reference_fixture_constants():
    rows = tier_s.encode_rows([3, 7, 11], [0, 1, 0], [0, 0, 1], [0, 0, 1], 8)
    np.testing.assert_allclose(rows, FIXTURE_ENCODER_ROWS, rtol=0, atol=1e-12)
    frame, stop, st = tier_s.decoder_step(tier_s.init_state(3, 8, 8), rows, 0.1)
    np.testing.assert_allclose(frame, FIXTURE_STEP_FRAME, rtol=0, atol=1e-12)
    assert stop == 0.0
    assert np.array_equal(st.attn_weights, np.full(3, 1.0 / 3.0))


def test_decoder_trace_matches_reference(golden_units):
    for i in range(3):
        ph, pw, pph, iph = golden_units[f"dec_in_{i}"]
        rows = tier_s.encode_rows(ph, pw, pph, iph, 8)
        st = tier_s.init_state(rows.shape[0], 8, 8)
        want = golden_units[f"dec_frames_{i}"]
        for k in range(want.shape[0]):
            frame, _, st = tier_s.decoder_step(st, rows, 0.1)
            np.testing.assert_allclose(frame, want[k], rtol=0, atol=1e-12)
            np.testing.assert_allclose(st.attn_weights, golden_units[f"dec_weights_{i}"][k], rtol=0, atol=1e-12)
        np.testing.assert_allclose(st.attn_weights_sum, golden_units[f"dec_wsum_{i}"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("ol", [4, 8])
def test_vocoder_splices_bit_exact(golden_units, ol):
    for j in range(5):
        key = f"voc_ol{ol}_{j}"
        mel, lens = golden_units[key + "_mel"], golden_units[key + "_lens"]
        st = tier_s.VocState(None, None, 0)
        got, offs, start = [], [], 0
        for k, m in enumerate(lens):
            s, off, st = tier_s.vocode_chunk(st, mel[start:start + m], k == len(lens) - 1, ol, 256)
            got.append(s), offs.append(off)
            start += m
        assert np.array_equal(np.array(offs), golden_units[key + "_offsets"])
        assert np.array_equal(np.array([g.size for g in got]), golden_units[key + "_counts"])
        assert np.array_equal(np.concatenate(got), golden_units[key + "_samples"])


def test_short_non_final_chunk_rejected():
    with pytest.raises(ValueError, match="overlap"):
        tier_s.vocode_chunk(tier_s.VocState(None, None, 0), np.zeros((3, 8)), False, 4, 256)


def test_decode_past_stop_rejected():
    rows = tier_s.encode_rows([1], [0], [0], [1], 8)
    mel, stop, st = tier_s.decode_chunk(tier_s.init_state(1, 8, 8), rows, 32, 0.1, 0.5)
    assert stop and mel.shape == (8, 8)
    with pytest.raises(ValueError, match="past stop"):
        tier_s.decode_chunk(st, rows, 32, 0.1, 0.5)


def test_synthesis_matches_reference(golden_synth, golden_frontend):
    for ol in (4, 8):
        for i, text in enumerate(golden_frontend["texts"]):
            fo = golden_frontend["outputs"][text]
            if len(fo["phonemes"]) > 60:  # long ones are covered on the GPU side
                continue
            chunks, _ = tier_s.synthesize(fo["phonemes"], fo["pw"], fo["pph"], fo["iph"],
                                          overlap_frames=ol)
            key = f"ol{ol}_{i}"
            assert [off for _, off in chunks] == list(golden_synth[key + "_offsets"])
            assert [s.size for s, _ in chunks] == list(golden_synth[key + "_counts"])
            np.testing.assert_allclose(np.concatenate([s for s, _ in chunks]),
                                       golden_synth[key + "_samples"], rtol=0, atol=1e-12)
