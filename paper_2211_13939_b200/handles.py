"""Device-resident values that cross the PipelineModules boundary.

The reference passes immutable numpy values between modules
(``EncodedFeatures``, ``DecoderState``, ``MelChunk``, ``VocoderState``;
``pkg/src/incrtts/acoustic.py:24-115``, ``vocoder.py:63-89``).  The GPU
modules keep those values in HBM and hand the scheduler *handles* that
duck-type the reference classes: host-visible counters are plain ints, the
arrays materialise lazily with a D2H copy only if someone reads them
(tests, debugging) -- the scheduler itself never does.

Value semantics are preserved without copying: every request owns ping-pong
state buffers in the ragged arena; a module call reads the input handle's
buffer and writes a buffer no live handle owns, so an old handle stays valid
(e.g. the per-item retry of ``_run_module``, ``scheduler.py:330-336``, or a
test that decodes the same state twice).  Buffers and regions are released
by weakref finalizers when the last handle of a request is dropped -- which
is how the modules learn about completions and failures the scheduler never
reports to them (``scheduler.py:490``).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import Any, Callable

import numpy as np
import torch


class _Buf:
    __slots__ = ("off", "size", "owner")

    def __init__(self, off: int, size: int):
        self.off, self.size, self.owner = off, size, None

    def free_for(self, taken: set) -> bool:
        return id(self) not in taken and (self.owner is None or self.owner() is None)


def _release_all(arena, regions, state_bufs, voc_bufs) -> None:
    # a finalizer: may run inside a cyclic collection on any thread, so the arena only queues it
    for off, size in regions:
        arena.release(off, size)
    for b in state_bufs + voc_bufs:
        arena.release(b.off, b.size)


class DeviceRequest:
    """Arena regions of one request; freed when the last handle goes away."""

    __slots__ = ("engine", "seq_len", "regions", "state_bufs", "voc_bufs", "extra", "__weakref__")

    def __init__(self, engine, seq_len: int):
        self.engine = engine
        self.seq_len = seq_len
        self.regions: list[tuple[int, int]] = []  # immutable regions, e.g. encoder memory
        self.state_bufs: list[_Buf] = []
        self.voc_bufs: list[_Buf] = []
        self.extra: dict[str, Any] = {}
        weakref.finalize(self, _release_all, engine.arena, self.regions, self.state_bufs,
                         self.voc_bufs)

    def add_region(self, size: int) -> int:
        off = self.engine.arena.alloc(size)
        self.regions.append((off, size))
        return off

    def claim(self, bufs: list[_Buf], size: int, taken: set) -> _Buf:
        """A buffer no live handle owns (and not used earlier in this call)."""
        for b in bufs:
            if b.size >= size and b.free_for(taken):
                taken.add(id(b))
                return b
        b = _Buf(self.engine.arena.alloc(size), size)
        bufs.append(b)
        taken.add(id(b))
        return b


class DeviceEncodedFeatures:
    """Duck-types ``EncodedFeatures`` (``acoustic.py:24-38``)."""

    __slots__ = ("req", "__weakref__")

    def __init__(self, req: DeviceRequest):
        self.req = req

    @property
    def seq_len(self) -> int:
        return self.req.seq_len

    @property
    def rows(self) -> np.ndarray:
        return self.req.engine.read_features(self.req)


class DeviceDecoderState:
    """Duck-types ``DecoderState`` (``acoustic.py:68-115``); arrays are lazy."""

    __slots__ = ("req", "buf", "frames_emitted", "target_frames", "_cache", "__weakref__")

    def __init__(self, req: DeviceRequest, buf: _Buf, frames_emitted: int, target_frames: int):
        self.req, self.buf = req, buf
        self.frames_emitted, self.target_frames = frames_emitted, target_frames
        self._cache = None
        buf.owner = weakref.ref(self)

    def _arrays(self) -> dict[str, np.ndarray]:
        if self._cache is None:
            self._cache = self.req.engine.read_state(self.req, self.buf)
        return self._cache

    def __getattr__(self, name):
        if name in ("last_frame", "attn_context", "attn_weights", "attn_weights_sum",
                    "attn_hidden", "attn_cell", "dec_hidden", "dec_cell"):
            return self._arrays()[name]
        raise AttributeError(name)


class DeviceMelChunk:
    """Duck-types ``MelChunk`` (``domain.py:181-199``): a view into a decode output.

    Built either from a tensor view, or lazily as row `row` of a [n][C][mel_dim] call output
    (the serving path: no per-item tensor slicing on the host); ``ptr`` / ``width`` /
    ``frame_count`` are plain ints either way.
    """

    __slots__ = ("_data", "_base", "_row", "_m", "_gate", "req", "__weakref__")

    def __init__(self, data, req: DeviceRequest | None):
        self._data, self._base, self._row, self._m, self._gate = data, None, 0, int(data.shape[0]), None
        self.req = req

    @classmethod
    def row_of(cls, base, row: int, frames: int, req: DeviceRequest | None, gate=None) -> "DeviceMelChunk":
        obj = cls.__new__(cls)
        obj._data, obj._base, obj._row, obj._m, obj._gate, obj.req = None, base, row, frames, gate, req
        return obj

    @property
    def data(self):
        if self._data is None:
            self._data = self._base[self._row, :self._m]
        return self._data

    @property
    def ptr(self) -> int:
        if self._data is not None:
            return self._data.data_ptr()
        return self._base.data_ptr() + self._row * self._base.stride(0) * self._base.element_size()

    @property
    def width(self) -> int:
        return int((self._data if self._data is not None else self._base).shape[-1])

    @property
    def gate_logits(self):
        """The chunk's stop-gate logits (Tier R computes them; stop itself is the frame counter)."""
        return None if self._gate is None else self._gate[self._row, :self._m]

    @property
    def frame_count(self) -> int:
        return self._m

    @property
    def frames(self) -> np.ndarray:
        if self.req is not None:
            self.req.engine.stream.synchronize()  # produced on the engine's stream
        else:
            torch.cuda.synchronize(self.data.device)
        arr = self.data.to("cpu").numpy().astype(np.float64)
        arr.setflags(write=False)
        return arr


class DeviceVocoderState:
    """Duck-types ``VocoderState`` (``vocoder.py:63-89``)."""

    __slots__ = ("req", "buf", "emitted_samples", "__weakref__")

    def __init__(self, req: DeviceRequest | None, buf: _Buf | None, emitted_samples: int):
        self.req, self.buf, self.emitted_samples = req, buf, emitted_samples
        if buf is not None:
            buf.owner = weakref.ref(self)

    @property
    def has_tail(self) -> bool:
        return self.buf is not None

    @property
    def mel_tail(self):
        return None if self.buf is None else self.req.engine.read_voc_state(self.req, self.buf)[0]

    @property
    def held_tail(self):
        return None if self.buf is None else self.req.engine.read_voc_state(self.req, self.buf)[1]


@dataclass(frozen=True)
class DecodeChunkResult:
    """``(mel, stop, state)`` as in ``acoustic.py:191-201``."""

    mel: Any
    stop: bool
    state: Any
