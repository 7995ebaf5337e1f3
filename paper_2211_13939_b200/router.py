"""Host router: request-sharded pools, one worker process per GPU (BASELINE config C4).

The reference serves everything from one loop (``SchedulerLoop``,
``pkg/src/incrtts/scheduler.py:548-597``); multi-GPU sharding is a non-goal
there (``SPEC.md:418``).  Requests never interact arithmetically (batch
transparency, ``SPEC.md:232``), so scaling out needs no collective: each
worker process owns one GPU, its own CUDA context, weight replica, request
pool and iteration loop; the router only moves text in and audio chunks out
over host IPC.

Data path per worker:

* text in: one ``mp.Queue`` (router -> worker);
* audio out: a shared-memory ring (``multiprocessing.shared_memory``) the
  worker writes samples into, plus ONE ``mp.Queue`` message per poll with the
  (request, offset-in-ring, length, sample offset) records and terminal events
  of every stream that moved -- no pickled audio, no thread per request.  The
  router copies the samples out and advances the ring's read cursor; a full
  ring back-pressures the worker's poller (never the serving loop).

Placement policies (deterministic):

* ``"least_frames"`` -- the worker with the fewest outstanding mel frames
  (target frames = frames_per_phoneme x phonemes, known from the frontend
  before admission), ties to the lowest index;
* ``"mod"`` -- request id modulo the worker count (parity runs).

Each worker records, per iteration, which requests its drain admitted, so a
worker's schedule can be replayed through the reference ``run_iteration``
and compared report by report (tests/test_router.py).  A worker that dies
fails its outstanding streams instead of leaving them open.
"""

from __future__ import annotations

import itertools
import multiprocessing as mp
import queue
import threading
import time
from dataclasses import dataclass, field
from multiprocessing import shared_memory

import numpy as np

from .domain import AudioChunk, PipelineConfig
from .frontend import default_lexicon, run_frontend
from .scheduler import ChunkStream, PoolClosed

_CHUNK, _DONE, _FAIL, _CANCEL = 0, 1, 2, 3
RING_BYTES = 128 << 20          # per worker: ~250 ms of audio at 275 QPS of 20 s requests
_HDR = 64                       # [0] write cursor (worker), [1] read cursor (router), bytes


@dataclass(frozen=True)
class WorkerSpec:
    """What a worker process builds: ``factory(lexicon, cfg, device)`` -> PipelineModules.

    ``factory`` is a "module:function" string so it survives the spawn
    start method (e.g. "paper_2211_13939_b200.modules:build_modules" with
    ``kwargs={"tier": "r"}``, or an oracle factory in CPU tests).
    ``warmup`` names a "module:function" called as ``fn(modules, cfg)`` in the
    worker before it reports ready (graph capture, allocator warm-up).
    """

    factory: str
    device: str | None
    cfg: PipelineConfig
    kwargs: dict = field(default_factory=dict)
    warmup: str | None = None


def _load(path: str):
    mod, fn = path.split(":")
    module = __import__(mod, fromlist=[fn])
    return getattr(module, fn)


class _RingWriter:
    """Worker side of the audio ring: contiguous records, wrap by skipping to offset 0."""

    def __init__(self, name: str):
        self.shm = shared_memory.SharedMemory(name=name)
        self.cur = np.ndarray((2,), dtype=np.int64, buffer=self.shm.buf[:16])
        self.data = self.shm.buf[_HDR:]
        self.cap = len(self.data)

    def put(self, arr: np.ndarray, stop: threading.Event) -> tuple[int, int]:
        """Copies `arr` into the ring -> (ring offset, end cursor); waits while the ring is full."""
        raw = arr.view(np.uint8).reshape(-1)
        n = raw.size
        if n > self.cap:
            raise ValueError("audio chunk larger than the router ring")
        head = int(self.cur[0])
        pos = head % self.cap
        if pos + n > self.cap:          # no split records: skip the tail of the ring
            head += self.cap - pos
            pos = 0
        while head + n - int(self.cur[1]) > self.cap:
            if stop.is_set():
                raise RuntimeError("router closed")
            time.sleep(0.0005)
        self.data[pos:pos + n] = raw
        self.cur[0] = head + n
        return pos, head + n

    def close(self) -> None:
        del self.cur, self.data
        self.shm.close()


def _worker_main(index: int, spec: WorkerSpec, ring_name: str, inbox: mp.Queue, outbox: mp.Queue) -> None:
    """Worker process: one pool + loop, one poller thread forwarding every stream's events."""
    if spec.device is not None and str(spec.device).startswith("cuda"):
        import torch
        torch.cuda.set_device(torch.device(spec.device))
    from .scheduler import CostModel, SchedulerLoop

    lex = default_lexicon()
    kwargs = dict(spec.kwargs)
    if spec.device is not None:
        kwargs["device"] = spec.device
    modules = _load(spec.factory)(lex, spec.cfg, **kwargs)
    if spec.warmup:
        _load(spec.warmup)(modules, spec.cfg)
    ring = _RingWriter(ring_name)
    admitted: list[list[int]] = []
    reports: list[tuple] = []
    local_to_global: dict[int, int] = {}
    first: dict[int, float] = {}          # gid -> perf_counter when its first chunk became visible
    live: list = []                       # (gid, stream) handed to the poller
    lock = threading.Lock()
    wake = threading.Event()
    stop_poll = threading.Event()

    def sink(rep) -> None:
        admitted.append([local_to_global[i] for i in rep.frontend_ids])
        reports.append((rep.step_index, [local_to_global[i] for i in rep.decoder_ids],
                        [local_to_global[i] for i in rep.completed_ids]))
        wake.set()

    def poller() -> None:
        pending: list = []
        while not (stop_poll.is_set() and not pending and not live):
            wake.wait(0.002)
            wake.clear()
            with lock:
                pending.extend(live)
                live.clear()
            records, keep = [], []
            for gid, stream in pending:
                try:
                    while True:
                        chunk = stream.get(timeout=0)
                        if chunk is None:
                            records.append((_DONE, gid, None))
                            break
                        samples = np.ascontiguousarray(chunk.samples)
                        pos, end = ring.put(samples, stop_poll)
                        records.append((_CHUNK, gid, (pos, samples.size, samples.dtype.str, chunk.sample_offset,
                                                      end, first.get(gid))))
                except queue.Empty:
                    keep.append((gid, stream))
                except Exception as exc:  # noqa: BLE001 -- forwarded to the client stream
                    records.append((_CANCEL if "cancelled" in str(exc) else _FAIL, gid, str(exc)))
            pending = keep
            if records:
                outbox.put((index, "batch", records))

    loop = SchedulerLoop(modules, CostModel.zero(), spec.cfg, report_sink=sink).start()
    poll_thread = threading.Thread(target=poller, name=f"router-poller-{index}", daemon=True)
    poll_thread.start()
    outbox.put((index, "ready", None))
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
        push = stream._push

        def timed_push(chunk, _push=push, _gid=gid):   # worker-side first-chunk time (CLOCK_MONOTONIC)
            if _gid not in first:
                first[_gid] = time.perf_counter()
            _push(chunk)

        stream._push = timed_push
        with lock:
            live.append((gid, stream))
        wake.set()
    loop.stop()
    stop_poll.set()
    wake.set()
    poll_thread.join(timeout=30)
    outbox.put((index, "exit", None, (admitted, reports)))
    ring.close()


class Router:
    """``submit(text) -> (request_id, ChunkStream)`` over N worker processes."""

    def __init__(self, specs: list[WorkerSpec], policy: str = "least_frames", ring_bytes: int = RING_BYTES,
                 ready_timeout: float = 900.0):
        if policy not in ("least_frames", "mod"):
            raise ValueError(f"unknown policy {policy!r}")
        self.policy = policy
        self.cfg = specs[0].cfg
        self._lex = default_lexicon()
        ctx = mp.get_context("spawn")
        self._outbox = ctx.Queue()
        self._inboxes = [ctx.Queue() for _ in specs]
        self._rings = [shared_memory.SharedMemory(create=True, size=_HDR + ring_bytes) for _ in specs]
        self._cursors = []
        for shm in self._rings:
            cur = np.ndarray((2,), dtype=np.int64, buffer=shm.buf[:16])
            cur[:] = 0
            self._cursors.append(cur)
        self._procs = [ctx.Process(target=_worker_main, args=(i, s, r.name, q, self._outbox), daemon=True)
                       for i, (s, r, q) in enumerate(zip(specs, self._rings, self._inboxes))]
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
        self.first_push: dict[int, float] = {}   # gid -> worker-side time its first chunk was visible
        self._ready = [threading.Event() for _ in specs]
        self._exited = [False] * len(specs)
        self.dead: list[int] = []
        self._closed = False
        self._pump = threading.Thread(target=self._drain, name="router-pump", daemon=True)
        self._pump.start()
        deadline = time.monotonic() + ready_timeout
        for i, ev in enumerate(self._ready):
            while not ev.wait(0.5):
                if i in self.dead or time.monotonic() > deadline:
                    self.close(timeout=5)
                    raise RuntimeError(f"router worker {i} failed to start")

    @property
    def workers(self) -> int:
        return len(self._procs)

    def _choose(self, gid: int, frames: int) -> int:
        live = [w for w in range(self.workers) if w not in self.dead]
        if not live:
            raise RuntimeError("no live router workers")
        if self.policy == "mod":
            w = (gid - 1) % self.workers
            return w if w in live else live[0]
        return min(live, key=lambda w: (self._outstanding[w], w))

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

    def _release(self, gid: int) -> ChunkStream | None:
        with self._lock:
            if gid not in self._frames:
                return None
            w, frames = self._frames.pop(gid)
            self._outstanding[w] -= frames
            return self._streams.pop(gid)

    def _fail_worker(self, w: int, why: str) -> None:
        """A worker died: fail every stream still placed on it."""
        self.dead.append(w)
        self._exited[w] = True
        with self._lock:
            gids = [g for g, (ww, _) in self._frames.items() if ww == w]
        for g in gids:
            s = self._release(g)
            if s is not None:
                s._fail(why)

    def _handle_batch(self, w: int, records: list) -> None:
        data = self._rings[w].buf[_HDR:]
        cur = self._cursors[w]
        for kind, gid, payload in records:
            if kind == _CHUNK:
                pos, count, dtype, offset, end, pushed = payload
                dt = np.dtype(dtype)
                samples = np.frombuffer(data, dtype=dt, count=count, offset=pos).copy()
                cur[1] = end
                with self._lock:
                    stream = self._streams.get(gid)
                if stream is not None:
                    self.first_push.setdefault(gid, pushed)
                    stream._push(AudioChunk.trusted(samples, offset))
            else:
                stream = self._release(gid)
                if stream is None:
                    continue
                if kind == _DONE:
                    stream._finish()
                elif kind == _FAIL:
                    stream._fail(payload)
                else:
                    stream._cancel()
        del data

    def _drain(self) -> None:
        while not all(self._exited):
            try:
                msg = self._outbox.get(timeout=0.2)
            except queue.Empty:
                msg = None
            if msg is not None:
                w, kind = msg[0], msg[1]
                if kind == "batch":
                    self._handle_batch(w, msg[2])
                elif kind == "ready":
                    self._ready[w].set()
                elif kind == "exit":
                    self.admissions[w], self.reports[w] = msg[3]
                    self._exited[w] = True
                continue
            for w, p in enumerate(self._procs):   # liveness: a worker that died without "exit"
                if not self._exited[w] and not p.is_alive():
                    self._fail_worker(w, f"router worker {w} died (exit code {p.exitcode})")

    def close(self, timeout: float = 60.0) -> None:
        if self._closed:
            return
        self._closed = True
        for w, q in enumerate(self._inboxes):
            if w not in self.dead:
                q.put(None)
        self._pump.join(timeout=timeout)
        for p in self._procs:
            p.join(timeout=5)
            if p.is_alive():
                p.terminate()
        self._cursors = []
        for shm in self._rings:
            try:
                shm.close()
                shm.unlink()
            except (FileNotFoundError, BufferError):
                pass

    def __enter__(self) -> "Router":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def gpu_router(n_gpus: int, cfg: PipelineConfig | None = None, tier: str = "r",
               policy: str = "least_frames", warmup: str | None = None, devices: list[str] | None = None,
               **kwargs) -> Router:
    """N worker processes, worker i on cuda:i (or devices[i]), GPU modules of the given tier."""
    cfg = cfg or PipelineConfig()
    devices = devices or [f"cuda:{i}" for i in range(n_gpus)]
    specs = [WorkerSpec("paper_2211_13939_b200.modules:build_modules", d, cfg, {"tier": tier, **kwargs}, warmup)
             for d in devices]
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
