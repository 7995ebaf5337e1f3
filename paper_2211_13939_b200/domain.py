"""Pipeline configuration and the value types that cross the module boundary.

Host-side mirror of the reference's domain layer (``pkg/src/incrtts/domain.py``):
same names, same field meanings, same validation errors, so code written
against the reference's ``PipelineConfig`` / ``MelChunk`` / ``AudioChunk``
runs unchanged here.  Nothing in this file touches the GPU.

Differences from the reference, all additive:

* ``PipelineConfig.tier`` is *not* a field (the reference CLI rejects unknown
  keys, ``pkg/src/incrtts/cli.py:37-39``); model tier and precision are
  chosen by the module factory instead (``paper_2211_13939_b200.modules``).
* ``AudioChunk.trusted`` / ``MelChunk`` handles let GPU modules hand back
  device-produced buffers without a second finite-check copy; the public
  constructors keep the reference's copy-and-validate behaviour
  (``domain.py:170-221``).
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np


class ConfigError(ValueError):
    """A configuration value violates an invariant (reference ``domain.py:15``)."""


@dataclass(frozen=True)
class PipelineConfig:
    """Knobs shared by every module (reference ``domain.py:55-91``).

    chunk_frames       mel frames per request per iteration (C)
    overlap_frames     frames re-synthesised at a chunk seam (O)
    hop_samples        audio samples per mel frame (H)
    sample_rate        Hz
    feature_dim        width of Tier-S stand-in vectors (Tier R ignores it)
    frames_per_phoneme stop counter: target = frames_per_phoneme * seq_len
    stop_threshold     stop fires when stop_value > threshold
    attention_penalty  Tier-S cumulative-attention penalty (lambda)
    """

    chunk_frames: int = 32
    overlap_frames: int = 4
    hop_samples: int = 256
    sample_rate: int = 22050
    feature_dim: int = 8
    frames_per_phoneme: int = 8
    stop_threshold: float = 0.5
    attention_penalty: float = 0.1

    @property
    def overlap_samples(self) -> int:
        return self.overlap_frames * self.hop_samples

    @property
    def chunk_seconds(self) -> float:
        return self.chunk_frames * self.hop_samples / self.sample_rate


# (predicate, message) pairs in the order the reference checks them
# (``domain.py:94-114``); the first failing rule raises.
_RULES = (
    (lambda c: c.chunk_frames >= 1, "chunk_frames must be >= 1"),
    (lambda c: c.overlap_frames >= 1, "overlap_frames must be >= 1"),
    (lambda c: c.overlap_frames < c.chunk_frames, "overlap must be < chunk"),
    (lambda c: c.hop_samples >= 1, "hop_samples must be >= 1"),
    (lambda c: c.sample_rate >= 1, "sample_rate must be >= 1"),
    (lambda c: c.feature_dim >= 1, "feature_dim must be >= 1"),
    (lambda c: c.frames_per_phoneme >= 1, "frames_per_phoneme must be >= 1"),
    (lambda c: 0.0 < c.stop_threshold < 1.0, "stop_threshold must lie strictly between 0 and 1"),
    (lambda c: c.attention_penalty >= 0.0, "attention_penalty must be >= 0"),
)


def validate_config(cfg: PipelineConfig) -> PipelineConfig:
    for ok, message in _RULES:
        if not ok(cfg):
            raise ConfigError(message)
    return cfg


def parse_kv(text: str) -> dict[str, str]:
    """``key = value`` lines; ``#`` comments; blank lines skipped (``domain.py:117-135``)."""
    out: dict[str, str] = {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        body = raw.partition("#")[0].strip()
        if not body:
            continue
        key, eq, value = body.partition("=")
        if not eq:
            raise ConfigError(f"line {lineno}: expected 'key = value', got {raw!r}")
        key = key.strip()
        if not key:
            raise ConfigError(f"line {lineno}: empty key")
        out[key] = value.strip()
    return out


_FIELD_TYPES = {f.name: f.type for f in fields(PipelineConfig)}


def config_keys() -> frozenset[str]:
    return frozenset(_FIELD_TYPES)


def config_from_mapping(mapping: dict[str, str]) -> PipelineConfig:
    """Typed, validated config from strings; foreign keys ignored (``domain.py:141-156``)."""
    kwargs = {}
    for name, ftype in _FIELD_TYPES.items():
        if name in mapping:
            conv = int if ftype in (int, "int") else float
            try:
                kwargs[name] = conv(mapping[name])
            except ValueError:
                raise ConfigError(f"config key {name}: cannot parse {mapping[name]!r}") from None
    return validate_config(PipelineConfig(**kwargs))


def load_config(path: str) -> PipelineConfig:
    with open(path, encoding="utf-8") as fh:
        return config_from_mapping(parse_kv(fh.read()))


def frozen_array(values, dtype=np.float64, ndim: int | None = None) -> np.ndarray:
    """Read-only finite copy (reference ``_frozen_array``, ``domain.py:170-178``)."""
    arr = np.array(values, dtype=dtype)
    if ndim is not None and arr.ndim != ndim:
        raise ValueError(f"expected a {ndim}-d array, got shape {arr.shape}")
    if not np.isfinite(arr).all():
        raise ValueError("array contains non-finite values")
    arr.setflags(write=False)
    return arr


_frozen_array = frozen_array


@dataclass(frozen=True)
class MelChunk:
    """``(frame_count, mel_dim)`` frames, >= 1 frame (``domain.py:181-199``)."""

    frames: np.ndarray

    def __post_init__(self) -> None:
        arr = frozen_array(self.frames, ndim=2)
        if arr.shape[0] < 1:
            raise ValueError("mel chunk needs at least one frame")
        object.__setattr__(self, "frames", arr)

    @property
    def frame_count(self) -> int:
        return int(self.frames.shape[0])


@dataclass(frozen=True)
class AudioChunk:
    """Samples plus absolute stream offset (``domain.py:202-221``)."""

    samples: np.ndarray
    sample_offset: int

    def __post_init__(self) -> None:
        object.__setattr__(self, "samples", frozen_array(self.samples, ndim=1))
        if self.sample_offset < 0:
            raise ValueError("sample_offset must be >= 0")

    @classmethod
    def trusted(cls, samples: np.ndarray, sample_offset: int) -> "AudioChunk":
        """Wraps a buffer a GPU module produced and already finite-checked on device.

        Skips the host copy + ``isfinite`` scan of the public constructor; the
        array is made read-only in place.
        """
        if sample_offset < 0:
            raise ValueError("sample_offset must be >= 0")
        obj = object.__new__(cls)
        samples.setflags(write=False)
        object.__setattr__(obj, "samples", samples)
        object.__setattr__(obj, "sample_offset", int(sample_offset))
        return obj

    @property
    def sample_count(self) -> int:
        return int(self.samples.shape[0])

    def pcm16(self) -> bytes:
        """16-bit little-endian PCM of the samples (the reference's ``pcm16_encode``,
        ``src/vocoder.py:146-149``, applied on the wire by ``src/server.py:176-200``).  GPU modules
        built with ``pcm16=True`` produce it on device in the splice pass, so the
        serving path skips the host conversion; otherwise it is computed here."""
        pre = self.__dict__.get("_pcm16")
        if pre is not None:
            return pre
        from .audio import pcm16_encode
        return pcm16_encode(self.samples)

    def wire_samples(self) -> str:
        """The reference server's ``"samples"`` field of a chunk frame: base64 of the 16-bit PCM
        (``encode_samples``, ``src/server.py:78-79``).  GPU modules built with ``wire_b64=True``
        produce it on device; otherwise it is computed here."""
        pre = self.__dict__.get("_b64")
        if pre is not None:
            return pre
        import base64
        return base64.b64encode(self.pcm16()).decode("ascii")
