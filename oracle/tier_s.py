"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the Tier-S (stand-in) arithmetic.

Numpy restatement of the reference ``incrtts`` stand-in models, used by
``tests/`` as the parity checker, by ``__graft_entry__.smoke()`` and by the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The product
path (``paper_2211_13939_b200``) never imports this package.

Parity pin: every function here is checked against golden vectors produced
by importing the reference itself (``tools/make_golden.py`` ->
``tests/golden/tier_s_*.npz``) and against the constants frozen in the
reference's own tests (``pkg/tests/test_domain.py:40-47``,
``pkg/tests/test_acoustic.py:32-47``).  Status: **pinned**.

Arithmetic order follows the reference op for op (numpy reductions over
axis 0 are sequential, the 8-wide row mean is numpy's pairwise block), so
encoder rows and vocoder samples are bit-identical to the reference; the
decoder's BLAS dot products may differ in the last ulp.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
TABLE_PHONEME, TABLE_PW, TABLE_PPH, TABLE_IPH = 0, 1, 2, 3


def splitmix64(keys: np.ndarray) -> np.ndarray:
    """SplitMix64 finalizer on uint64 arrays (reference ``domain.py:22-30``)."""
    z = np.asarray(keys, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def seeded_vectors(table_id: int, tokens, dim: int) -> np.ndarray:
    """Rows ``seeded_vector(table_id, tok, dim)`` for each token (``domain.py:33-52``).

    Key = table in bits 56-63, token in bits 16-55, component in bits 0-15;
    value = top 53 hash bits mapped onto [-1, 1).
    """
    tok = np.asarray(tokens, dtype=np.uint64).reshape(-1, 1) & np.uint64(0xFFFFFFFFFF)
    comp = np.arange(dim, dtype=np.uint64).reshape(1, -1) & np.uint64(0xFFFF)
    keys = (np.uint64(table_id & 0xFF) << np.uint64(56)) | (tok << np.uint64(16)) | comp
    h = splitmix64(keys)
    return (h >> np.uint64(11)).astype(np.float64) / float(1 << 53) * 2.0 - 1.0


def seeded_vector(table_id: int, token_id: int, dim: int) -> np.ndarray:
    if dim < 1:
        raise ValueError("dim must be >= 1")
    return seeded_vectors(table_id, [token_id], dim)[0]


def embed_sum(phonemes, pw, pph, iph, dim: int) -> np.ndarray:
    """E_all[t] = ((phoneme + pw) + pph) + iph, paper Eq. 1 (``acoustic.py:52-59``)."""
    return (seeded_vectors(TABLE_PHONEME, phonemes, dim) + seeded_vectors(TABLE_PW, pw, dim)
            + seeded_vectors(TABLE_PPH, pph, dim) + seeded_vectors(TABLE_IPH, iph, dim))


def encode_rows(phonemes, pw, pph, iph, dim: int) -> np.ndarray:
    """F[t] = (E[t] + mean(E[:t+1]) + mean(E[t:])) / 3 (``acoustic.py:41-65``).

    Same slice means as the reference (O(L^2)), so rows are bit-identical.
    """
    summed = embed_sum(phonemes, pw, pph, iph, dim)
    n = summed.shape[0]
    rows = np.empty_like(summed)
    for t in range(n):
        rows[t] = (summed[t] + summed[: t + 1].mean(axis=0) + summed[t:].mean(axis=0)) / 3.0
    return rows


@dataclass
class DecState:
    """The eight Eq.-2 tensors plus counters (``acoustic.py:68-115``)."""

    last_frame: np.ndarray
    attn_context: np.ndarray
    attn_weights: np.ndarray
    attn_weights_sum: np.ndarray
    attn_hidden: np.ndarray
    attn_cell: np.ndarray
    dec_hidden: np.ndarray
    dec_cell: np.ndarray
    frames_emitted: int
    target_frames: int


def init_state(seq_len: int, dim: int, frames_per_phoneme: int) -> DecState:
    """Zero state, target = frames_per_phoneme * L (``acoustic.py:118-133``)."""
    z = np.zeros(dim)
    return DecState(z, z, np.zeros(seq_len), np.zeros(seq_len), z, z, z, z, 0,
                    frames_per_phoneme * seq_len)


def _cell(x2: np.ndarray, hidden: np.ndarray, cell: np.ndarray):
    """Fold halves, C' = tanh(.5C + .5fold + .25H), H' = tanh(C') (``acoustic.py:136-146``)."""
    fold = x2.reshape(-1, hidden.shape[0]).sum(axis=0)
    c = np.tanh(0.5 * cell + 0.5 * fold + 0.25 * hidden)
    return np.tanh(c), c


def decoder_step(s: DecState, rows: np.ndarray, penalty: float):
    """One frame, Eq.-2 order (``acoustic.py:154-188``); returns (frame, stop_value, state)."""
    if s.attn_weights.shape[0] != rows.shape[0]:
        raise ValueError("decoder state does not match encoded features")
    h_att, c_att = _cell(np.concatenate([np.tanh(s.last_frame), s.attn_context]),
                         s.attn_hidden, s.attn_cell)
    scores = rows @ h_att - penalty * s.attn_weights_sum
    e = np.exp(scores - scores.max())
    w = e / e.sum()
    ctx = w @ rows
    h_dec, c_dec = _cell(np.concatenate([h_att, ctx]), s.dec_hidden, s.dec_cell)
    frame = np.tanh(h_dec + ctx)
    n = s.frames_emitted + 1
    stop = 1.0 if n >= s.target_frames else 0.0
    return frame, stop, DecState(frame, ctx, w, s.attn_weights_sum + w, h_att, c_att,
                                 h_dec, c_dec, n, s.target_frames)


def decode_chunk(s: DecState, rows: np.ndarray, chunk_frames: int, penalty: float,
                 stop_threshold: float):
    """<= C steps, truncated at the stop gate (``acoustic.py:204-219``).

    Returns (mel[m, D], stopped, state).
    """
    if s.frames_emitted >= s.target_frames:
        raise ValueError("decode past stop")
    frames = []
    for _ in range(chunk_frames):
        frame, stop_value, s = decoder_step(s, rows, penalty)
        frames.append(frame)
        if stop_value > stop_threshold:
            return np.stack(frames), True, s
    return np.stack(frames), False, s


def generate(mel: np.ndarray, hop: int) -> np.ndarray:
    """Stand-in G: each frame's mean repeated ``hop`` times (``vocoder.py:52-60``)."""
    return np.repeat(mel.mean(axis=1), hop)


def crossfade(length: int) -> tuple[np.ndarray, np.ndarray]:
    """(fade_in, fade_out) = (sin, cos)(pi/2 (k+.5)/S) (``vocoder.py:35-44``)."""
    theta = (np.pi / 2.0) * ((np.arange(length, dtype=np.float64) + 0.5) / length)
    return np.sin(theta), np.cos(theta)


@dataclass
class VocState:
    mel_tail: np.ndarray | None
    held_tail: np.ndarray | None
    emitted_samples: int = 0


def vocode_chunk(state: VocState, mel: np.ndarray, is_last: bool, overlap_frames: int,
                 hop: int, gen=generate):
    """Splice + equal-power fuse + hold-back (``vocoder.py:92-136``, paper Eq. 3-4).

    Returns (samples, sample_offset, new_state).  ``gen(mel, hop)`` is the
    vocoder G; Tier R passes HiFi-GAN here.
    """
    S = overlap_frames * hop
    if not is_last and mel.shape[0] < overlap_frames:
        raise ValueError("non-final chunk shorter than the overlap window")
    offset = state.emitted_samples
    if state.mel_tail is None:
        samples = gen(mel, hop)
        if is_last:
            return samples, offset, VocState(None, None, offset + samples.size)
        if samples.size <= S:
            raise ValueError("non-final chunk shorter than the overlap window")
        out = samples[:-S]
        return out, offset, VocState(mel[-overlap_frames:], samples[-S:], offset + out.size)
    fade_in, fade_out = crossfade(S)
    samples = gen(np.concatenate([state.mel_tail, mel]), hop)
    fused = fade_in * samples[:S] + fade_out * state.held_tail
    if is_last:
        out = np.concatenate([fused, samples[S:]])
        return out, offset, VocState(None, None, offset + out.size)
    out = np.concatenate([fused, samples[S:-S]])
    return out, offset, VocState(mel[-overlap_frames:], samples[-S:], offset + out.size)


def synthesize(phonemes, pw, pph, iph, *, dim=8, frames_per_phoneme=8, chunk_frames=32,
               overlap_frames=4, hop=256, penalty=0.1, stop_threshold=0.5):
    """Single-request incremental synthesis (``synthesis.py:33-48``).

    Returns (list of (samples, offset), mel [F, D]).
    """
    rows = encode_rows(phonemes, pw, pph, iph, dim)
    s = init_state(rows.shape[0], dim, frames_per_phoneme)
    v = VocState(None, None, 0)
    chunks, mels = [], []
    while True:
        mel, stop, s = decode_chunk(s, rows, chunk_frames, penalty, stop_threshold)
        mels.append(mel)
        samples, off, v = vocode_chunk(v, mel, stop, overlap_frames, hop)
        chunks.append((samples, off))
        if stop:
            return chunks, np.concatenate(mels)
