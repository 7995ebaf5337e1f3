"""TEST INFRASTRUCTURE ONLY -- oracle arithmetic behind the PipelineModules boundary.

``cpu_modules(lexicon, cfg)`` returns a :class:`PipelineModules` whose
encoder / decoder / vocoder callables are the numpy Tier-S oracle
(``oracle/tier_s.py``), i.e. a CPU restatement of the reference's
``build_modules`` (``pkg/src/incrtts/scheduler.py:266-282``).  Used by the
parity tests (schedules, batch transparency) and by ``bench.py``'s
reference arm.  Never imported by the product package.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2211_13939_b200.domain import AudioChunk, MelChunk, PipelineConfig
from paper_2211_13939_b200.scheduler import PipelineModules, frontend_module

from . import tier_s


@dataclass(frozen=True)
class Encoded:
    rows: np.ndarray

    @property
    def seq_len(self) -> int:
        return int(self.rows.shape[0])


@dataclass(frozen=True)
class DecodeResult:
    mel: MelChunk
    stop: bool
    state: tier_s.DecState


def cpu_modules(lexicon, cfg: PipelineConfig) -> PipelineModules:
    dim = cfg.feature_dim

    def encoder(fos):
        out = []
        for fo in fos:
            rows = tier_s.encode_rows(fo.phonemes, fo.pw, fo.pph, fo.iph, dim)
            out.append((Encoded(rows), tier_s.init_state(rows.shape[0], dim, cfg.frames_per_phoneme)))
        return out

    def decoder(pairs):
        out = []
        for state, enc in pairs:
            mel, stop, new = tier_s.decode_chunk(state, enc.rows, cfg.chunk_frames,
                                                 cfg.attention_penalty, cfg.stop_threshold)
            out.append(DecodeResult(MelChunk(mel), stop, new))
        return out

    def vocoder(triples):
        out = []
        for state, mel, is_last in triples:
            st = tier_s.VocState(state.mel_tail, state.held_tail, state.emitted_samples)
            samples, off, new = tier_s.vocode_chunk(st, mel.frames, is_last, cfg.overlap_frames,
                                                    cfg.hop_samples)
            out.append((AudioChunk(samples, off), new))
        return out

    mods = PipelineModules(frontend_module(lexicon), encoder, decoder, vocoder)

    def decoder_steps(triples):   # step-granular admission: <= limit steps of the current chunk
        out = []
        for state, enc, limit in triples:
            mel, stop, new = tier_s.decode_chunk(state, enc.rows, min(int(limit), cfg.chunk_frames),
                                                 cfg.attention_penalty, cfg.stop_threshold)
            out.append(DecodeResult(MelChunk(mel), stop, new))
        return out

    object.__setattr__(mods, "decoder_steps", decoder_steps)
    object.__setattr__(mods, "concat_mels", lambda parts: MelChunk(np.concatenate([p.frames for p in parts], 0)))
    return mods


def cpu_modules_r(lexicon, cfg: PipelineConfig, weights, deadline: float | None = None) -> PipelineModules:
    """Tier-R oracle (torch-CPU fp32 Tacotron2 + HiFi-GAN) behind the same boundary.

    Batched calls are plain per-item loops, like the reference's
    ``encode_batch`` / ``decode_chunk_batch`` / ``vocode_batch``.
    """
    import time

    from . import tier_r

    def check():
        if deadline is not None and time.perf_counter() > deadline:
            raise TimeoutError("cpu baseline time budget exhausted")

    def encoder(fos):
        out = []
        for fo in fos:
            check()
            mem, pm = tier_r.encode(weights, fo.phonemes, fo.pw, fo.pph, fo.iph)
            out.append((EncodedR(mem, pm), tier_r.init_state(mem.shape[0], cfg.frames_per_phoneme)))
        return out

    def decoder(pairs):
        out = []
        for state, enc in pairs:
            check()
            mel, stop, new, _ = tier_r.decode_chunk(weights, state, enc.memory, enc.pm, cfg.chunk_frames)
            out.append(DecodeResult(MelChunk(mel.numpy()), stop, new))
        return out

    def vocoder(triples):
        out = []
        for state, mel, is_last in triples:
            check()
            st = tier_s.VocState(state.mel_tail, state.held_tail, state.emitted_samples)
            samples, off, new = tier_r.vocode_chunk(weights, st, mel.frames, is_last, cfg.overlap_frames,
                                                    cfg.hop_samples)
            out.append((AudioChunk(samples, off), new))
        return out

    return PipelineModules(frontend_module(lexicon), encoder, decoder, vocoder)


@dataclass(frozen=True)
class EncodedR:
    memory: object
    pm: object

    @property
    def seq_len(self) -> int:
        return int(self.memory.shape[0])


def crashing_modules(lexicon, cfg: PipelineConfig) -> PipelineModules:
    """Tier-S oracle modules whose decoder kills the process on a text that maps to >= 40
    phonemes (router liveness tests: a worker dying mid-stream)."""
    import os

    base = cpu_modules(lexicon, cfg)

    def decoder(pairs):
        if any(enc.seq_len >= 40 for _, enc in pairs):
            os._exit(3)
        return base.decoder_batch(pairs)

    return PipelineModules(base.frontend_batch, base.encoder_batch, decoder, base.vocoder_batch)
