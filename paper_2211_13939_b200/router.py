"""Host router: request-sharded pools, one worker process per GPU (BASELINE config C4).

The reference serves everything from one loop (``SchedulerLoop``,
``pkg/src/incrtts/scheduler.py:548-597``); multi-GPU sharding is a non-goal
there (``SPEC.md:418``).  Requests never interact arithmetically (batch
transparency, ``SPEC.md:232``), so scaling out needs no collective: each
worker process owns one GPU, its own CUDA context, weight replica, request
pool and iteration loop; the router only moves text in and audio chunks out
over host IPC.

Placement policies (deterministic):

* ``"least_frames"`` -- the worker with the fewest outstanding mel frames
  (target frames = frames_per_phoneme x phonemes, known from the frontend
  before admission), ties to the lowest index;
* ``"mod"`` -- request id modulo the worker count (parity runs).

Each worker records, per iteration, which requests its drain admitted, so a
worker's schedule can be replayed through the reference ``run_iteration``
and compared report by report (tests/test_router.py).
"""

from __future__ import annotations

import itertools
import multiprocessing as mp
import queue
import threading
import time
from dataclasses import dataclass

import numpy as np

from .domain import AudioChunk, PipelineConfig
from .frontend import default_lexicon, run_frontend
from .scheduler import ChunkStream, PoolClosed

_CHUNK, _DONE, _FAIL, _CANCEL, _REPORT = "chunk", "done", "fail", "cancel", "report"


@dataclass(frozen=True)
class WorkerSpec:
    """What a worker process builds: ``factory(lexicon, cfg, device)`` -> PipelineModules.

    ``factory`` is a "module:function" string so it survives the spawn
    start method (e.g. "paper_2211_13939_b200.modules:build_modules" with
    ``kwargs={"tier": "r"}``, or an oracle factory in CPU tests).
    """

    factory: str
    device: str | None
    cfg: PipelineConfig
    kwargs: dict


def _load(path: str):
    mod, fn = path.split(":")
    module = __import__(mod, fromlist=[fn])
    return getattr(module, fn)


def _worker_main(index: int, spec: WorkerSpec, inbox: mp.Queue, outbox: mp.Queue) -> None:
    """Worker process: one pool + loop; forwards every chunk / terminal event to the router."""
    from .scheduler import CostModel, SchedulerLoop

    lex = default_lexicon()
    kwargs = dict(spec.kwargs)
    if spec.device is not None:
        kwargs["device"] = spec.device
    modules = _load(spec.factory)(lex, spec.cfg, **kwargs)
    admitted: list[list[int]] = []
    local_to_global: dict[int, int] = {}

    def sink(rep) -> None:
        admitted.append([local_to_global[i] for i in rep.frontend_ids])
        outbox.put((index, _REPORT, None, (rep.step_index, [local_to_global[i] for i in rep.decoder_ids],
                                            [local_to_global[i] for i in rep.completed_ids])))

    loop = SchedulerLoop(modules, CostModel.zero(), spec.cfg, report_sink=sink).start()
    forwarders: list[threading.Thread] = []

    def forward(gid: int, stream: ChunkStream) -> None:
        try:
            for chunk in stream:
                arr = np.ascontiguousarray(chunk.samples)
                outbox.put((index, _CHUNK, gid, (arr.tobytes(), arr.dtype.str, chunk.sample_offset)))
            outbox.put((index, _DONE, gid, None))
        except Exception as exc:  # noqa: BLE001 -- forwarded to the client stream
            kind = _CANCEL if "cancelled" in str(exc) else _FAIL
            outbox.put((index, kind, gid, str(exc)))

    submitted = 0
    while True:
        msg = inbox.get()
        if msg is None:
            break
        gid, text = msg
        submitted += 1
        local_to_global[submitted] = gid  # pool ids are 1, 2, ... in submit order; map before admission
        lid, stream = loop.submit(text)
        assert lid == submitted
        t = threading.Thread(target=forward, args=(gid, stream), daemon=True)
        t.start()
        forwarders.append(t)
    loop.stop()
    for t in forwarders:
        t.join(timeout=5)
    outbox.put((index, "exit", None, admitted))


class Router:
    """``submit(text) -> (request_id, ChunkStream)`` over N worker processes."""

    def __init__(self, specs: list[WorkerSpec], policy: str = "least_frames"):
        if policy not in ("least_frames", "mod"):
            raise ValueError(f"unknown policy {policy!r}")
        self.policy = policy
        self.cfg = specs[0].cfg
        self._lex = default_lexicon()
        ctx = mp.get_context("spawn")
        self._outbox = ctx.Queue()
        self._inboxes = [ctx.Queue() for _ in specs]
        self._procs = [ctx.Process(target=_worker_main, args=(i, s, q, self._outbox), daemon=True)
                       for i, (s, q) in enumerate(zip(specs, self._inboxes))]
        for p in self._procs:
            p.start()
        self._ids = itertools.count(1)
        self._lock = threading.Lock()
        self._streams: dict[int, ChunkStream] = {}
        self._outstanding = [0] * len(specs)
        self._frames: dict[int, tuple[int, int]] = {}   # gid -> (worker, frames)
        self.placement: dict[int, int] = {}
        self.reports: list[list] = [[] for _ in specs]
        self.admissions: list[list[list[int]] | None] = [None] * len(specs)
        self._closed = False
        self._pump = threading.Thread(target=self._drain, name="router-pump", daemon=True)
        self._pump.start()

    @property
    def workers(self) -> int:
        return len(self._procs)

    def _choose(self, gid: int, frames: int) -> int:
        if self.policy == "mod":
            return (gid - 1) % self.workers
        return min(range(self.workers), key=lambda w: (self._outstanding[w], w))

    def submit(self, text: str) -> tuple[int, ChunkStream]:
        if self._closed:
            raise PoolClosed("router is shut down")
        if not text:
            raise ValueError("empty input")
        frames = self.cfg.frames_per_phoneme * run_frontend(text, self._lex).seq_len
        with self._lock:
            gid = next(self._ids)
            w = self._choose(gid, frames)
            stream = ChunkStream(gid)
            self._streams[gid] = stream
            self._outstanding[w] += frames
            self._frames[gid] = (w, frames)
            self.placement[gid] = w
        self._inboxes[w].put((gid, text))
        return gid, stream

    def _release(self, gid: int) -> ChunkStream:
        with self._lock:
            w, frames = self._frames.pop(gid)
            self._outstanding[w] -= frames
            return self._streams.pop(gid)

    def _drain(self) -> None:
        exited = 0
        while exited < self.workers:
            w, kind, gid, payload = self._outbox.get()
            if kind == _CHUNK:
                samples, dtype, offset = payload
                with self._lock:
                    stream = self._streams.get(gid)
                if stream is not None:
                    stream._push(AudioChunk.trusted(np.frombuffer(samples, dtype=np.dtype(dtype)).copy(), offset))
            elif kind == _DONE:
                self._release(gid)._finish()
            elif kind == _FAIL:
                self._release(gid)._fail(payload)
            elif kind == _CANCEL:
                self._release(gid)._cancel()
            elif kind == _REPORT:
                self.reports[w].append(payload)
            elif kind == "exit":
                self.admissions[w] = payload
                exited += 1

    def close(self, timeout: float = 60.0) -> None:
        if self._closed:
            return
        self._closed = True
        for q in self._inboxes:
            q.put(None)
        self._pump.join(timeout=timeout)
        for p in self._procs:
            p.join(timeout=5)

    def __enter__(self) -> "Router":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def gpu_router(n_gpus: int, cfg: PipelineConfig | None = None, tier: str = "r",
               policy: str = "least_frames") -> Router:
    """N worker processes, worker i on cuda:i, GPU modules of the given tier."""
    cfg = cfg or PipelineConfig()
    specs = [WorkerSpec("paper_2211_13939_b200.modules:build_modules", f"cuda:{i}", cfg, {"tier": tier})
             for i in range(n_gpus)]
    return Router(specs, policy)


def wait_all(streams, timeout: float = 120.0) -> list[list[AudioChunk]]:
    """Collects every stream (helper for tests / examples)."""
    out, deadline = [], time.time() + timeout
    for s in streams:
        chunks = []
        while True:
            c = s.get(timeout=max(0.1, deadline - time.time()))
            if c is None:
                break
            chunks.append(c)
        out.append(chunks)
    return out
