"""Vocoder carry-over state, cross-fade ramps and PCM helpers (host side).

Mirrors the host-visible parts of the reference vocoder
(``pkg/src/incrtts/vocoder.py``): the ``VocoderState`` value the scheduler
constructs for every new request (``scheduler.py:448``), the equal-power
ramps of Eq. 3 (``vocoder.py:21-49``) and PCM16/WAV I/O
(``vocoder.py:146-165``).  The per-chunk splice itself runs on the GPU
(``csrc/tier_s.cu`` / ``csrc/hifigan.cu``); GPU modules return
``DeviceVocoderState`` handles that duck-type this class.
"""

from __future__ import annotations

import wave
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .domain import frozen_array

PCM_SCALE = 32767


@dataclass(frozen=True)
class VocoderState:
    """``mel_tail`` (O frames) + ``held_tail`` (S samples) + emitted count.

    Both tails are None before the first chunk and after the last
    (reference ``vocoder.py:63-89``).
    """

    mel_tail: np.ndarray | None
    held_tail: np.ndarray | None
    emitted_samples: int = 0

    def __post_init__(self) -> None:
        if (self.mel_tail is None) != (self.held_tail is None):
            raise ValueError("mel_tail and held_tail must be set together")
        if self.mel_tail is not None:
            object.__setattr__(self, "mel_tail", frozen_array(self.mel_tail, ndim=2))
            object.__setattr__(self, "held_tail", frozen_array(self.held_tail, ndim=1))
        if self.emitted_samples < 0:
            raise ValueError("emitted_samples must be >= 0")

    @classmethod
    def initial(cls) -> "VocoderState":
        return cls(None, None, 0)


@dataclass(frozen=True)
class CrossfadeCurve:
    """``fade_in[k]**2 + fade_out[k]**2 == 1`` ramps (``vocoder.py:21-32``)."""

    fade_in: np.ndarray
    fade_out: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "fade_in", frozen_array(self.fade_in, ndim=1))
        object.__setattr__(self, "fade_out", frozen_array(self.fade_out, ndim=1))
        if self.fade_in.shape != self.fade_out.shape:
            raise ValueError("fade ramps must have equal length")


def crossfade_curve(length: int) -> CrossfadeCurve:
    """Window-centred sin/cos ramps, theta_k = pi/2 (k+0.5)/length (``vocoder.py:35-44``)."""
    if length < 1:
        raise ValueError("crossfade length must be >= 1")
    theta = (np.arange(length, dtype=np.float64) + 0.5) / length * (np.pi / 2.0)
    return CrossfadeCurve(np.sin(theta), np.cos(theta))


@lru_cache(maxsize=None)
def cached_curve(length: int) -> CrossfadeCurve:
    return crossfade_curve(length)


def pcm16_encode(samples: np.ndarray) -> bytes:
    """Clamp to [-1, 1], scale by 32767, round half-to-even, little-endian int16."""
    x = np.clip(np.asarray(samples, dtype=np.float64), -1.0, 1.0)
    return np.round(x * PCM_SCALE).astype("<i2").tobytes()


def pcm16_decode(data: bytes) -> np.ndarray:
    if len(data) % 2:
        raise ValueError("PCM payload has odd byte length")
    return np.frombuffer(data, dtype="<i2").astype(np.float64) / PCM_SCALE


def write_wav(path: str, samples: np.ndarray, sample_rate: int) -> None:
    with wave.open(path, "wb") as fh:
        fh.setnchannels(1)
        fh.setsampwidth(2)
        fh.setframerate(sample_rate)
        fh.writeframes(pcm16_encode(samples))
