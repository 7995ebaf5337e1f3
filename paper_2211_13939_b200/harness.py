"""Load harness: traces, a timed serving run, latency records and percentiles.

Mirrors the reference harness (``pkg/src/incrtts/harness.py``): evenly
spaced traces (``make_trace``, ``:97-118``), client-side FCL / LCL / RTF
(``LatencyRecord``, ``:121-152``), nearest-rank percentiles (``:267-275``)
-- and adds what the B200 measurement needs: Poisson
arrivals, per-request timestamps taken both where the chunk becomes
visible on the stream (server boundary) and where a client thread
receives it, and an iteration-indexed timing window so a bench can time
exactly K scheduler iterations after W warm-up iterations.
"""

from __future__ import annotations

import collections
import math
import queue
import random
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

from .frontend import Lexicon, default_lexicon, default_texts
from .scheduler import CostModel, IterationReport, PipelineModules, RequestCancelled, SchedulerLoop, _wait_until


@dataclass(frozen=True)
class TimedRequest:
    send_at: float
    text: str
    text_class: str = "random"


def make_trace(qps: int, duration_seconds: float, text_class: str = "mixed", seed: int = 0,
               fixtures: dict | None = None) -> list[TimedRequest]:
    """Evenly spaced trace, request i at i/qps (reference ``make_trace``)."""
    fixtures = default_texts() if fixtures is None else fixtures
    classes = ("short", "medium", "long") if text_class == "mixed" else (text_class,)
    rng = random.Random(seed)
    out = []
    for i in range(int(qps * duration_seconds)):
        cls = rng.choice(classes) if text_class == "mixed" else text_class
        texts = fixtures[cls]
        out.append(TimedRequest(i / qps, texts[i % len(texts)], cls))
    return out


def random_text(rng: random.Random, lo: int, hi: int, lexicon: Lexicon | None = None) -> str:
    """U{lo..hi} characters drawn from the single-character lexicon entries."""
    lex = lexicon or default_lexicon()
    singles = sorted(c for c in lex.phrase_to_pinyin if len(c) == 1)
    return "".join(rng.choice(singles) for _ in range(rng.randint(lo, hi)))


def poisson_trace(qps: float, duration_seconds: float, lo: int = 20, hi: int = 200, seed: int = 0,
                  lexicon: Lexicon | None = None) -> list[TimedRequest]:
    """Exponential inter-arrivals at rate ``qps``; lengths U{lo..hi} chars."""
    rng = random.Random(seed)
    t, out = 0.0, []
    while True:
        t += rng.expovariate(qps)
        if t >= duration_seconds:
            return out
        out.append(TimedRequest(t, random_text(rng, lo, hi, lexicon)))


@dataclass
class RequestTiming:
    request_id: int
    text: str
    send_time: float
    first_push: float | None = None      # chunk visible on the ChunkStream (server boundary)
    first_recv: float | None = None      # client thread received it
    last_recv: float | None = None
    samples: int = 0
    chunks: int = 0
    error: str | None = None
    cancelled: bool = False              # cancelled by the server's shutdown (after the window)
    done: bool = False

    @property
    def fcl(self) -> float | None:
        return None if self.first_push is None else self.first_push - self.send_time

    @property
    def fcl_client(self) -> float | None:
        return None if self.first_recv is None else self.first_recv - self.send_time

    @property
    def lcl(self) -> float | None:
        return None if self.last_recv is None else self.last_recv - self.send_time


def nearest_rank(values, percentile: float) -> float:
    if not values:
        raise ValueError("no values")
    ordered = sorted(values)
    return ordered[max(1, math.ceil(percentile / 100.0 * len(ordered))) - 1]


@dataclass
class ServeRun:
    """Result of :func:`serve`: per-request timings plus per-iteration end times."""

    timings: list[RequestTiming]
    iteration_end: list[float] = field(default_factory=list)
    reports: list[IterationReport] = field(default_factory=list)
    window: tuple[float, float] | None = None


def serve(modules: PipelineModules, cfg, trace: list[TimedRequest], *, warmup_iters: int = 3,
          warmup_seconds: float = 0.0, timed_iters: int | None = None, drain_seconds: float = 30.0,
          on_window=None, max_clients: int = 4096, sample_rate: int = 22050,
          tail_seconds: float = 120.0, timed_seconds: float | None = None,
          consumers: bool = True, client: str = "poller", admission: str = "iteration",
          sub_steps: int = 8) -> ServeRun:
    """Plays ``trace`` against a fresh SchedulerLoop and records every request.

    The timed window is iterations ``[w, w + timed_iters)`` where ``w`` is the
    first iteration index >= ``warmup_iters`` that starts after
    ``warmup_seconds``.  ``on_window(kind, iteration_index)`` is called from
    the loop thread at the window's start and end (bench hooks: CUDA events,
    clock sampling).  Submissions continue until every request sent inside
    the window has finished (or ``drain_seconds`` passed), so the load seen
    by the measured requests stays at the trace rate.
    """
    run = ServeRun(timings=[])
    lock = threading.Lock()
    state = {"start_idx": None, "end_idx": None}
    origin = time.perf_counter()

    def sink(rep: IterationReport) -> None:
        now = time.perf_counter()
        run.iteration_end.append(now)
        run.reports.append(rep)
        i = len(run.iteration_end)  # iterations completed so far == index of the next iteration
        if state["start_idx"] is None and i >= warmup_iters and now - origin >= warmup_seconds:
            state["start_idx"] = i
            run.window = (now, None)
            if on_window:
                on_window("start", i)
        elif (state["start_idx"] is not None and state["end_idx"] is None
              and ((timed_iters is not None and i >= state["start_idx"] + timed_iters)
                   or (timed_seconds is not None and now - run.window[0] >= timed_seconds))):
            state["end_idx"] = i
            run.window = (run.window[0], now)
            if on_window:
                on_window("end", i)

    wake = threading.Event()
    # streams that received something since the poller last looked: the loop thread appends on
    # every push / terminal event (deque.append is atomic), so the poller touches only those --
    # like a client woken per message -- instead of polling every open stream (at 240 live
    # requests that polling cost ~25 % of the GIL and slowed the serving loop)
    dirty: collections.deque = collections.deque()

    def sink_and_wake(rep: IterationReport) -> None:
        sink(rep)
        wake.set()

    loop = SchedulerLoop(modules, CostModel.zero(), cfg, report_sink=sink_and_wake if client == "poller" else sink,
                         admission=admission, sub_steps=sub_steps)
    stop_poll = threading.Event()

    def poller() -> None:
        while True:
            wake.wait(0.002)
            wake.clear()
            touched = {}
            while dirty:
                rec, stream = dirty.popleft()
                touched[id(rec)] = (rec, stream)
            for rec, stream in touched.values():
                if rec.done:
                    continue
                try:
                    while True:
                        chunk = stream.get(timeout=0)
                        now = time.perf_counter()
                        if chunk is None:
                            rec.done = True
                            break
                        if rec.first_recv is None:
                            rec.first_recv = now
                        rec.last_recv = now
                        rec.samples += chunk.sample_count
                        rec.chunks += 1
                except queue.Empty:
                    pass
                except RequestCancelled:   # the loop stopped after the window: not a failure
                    rec.cancelled = True
                    rec.done = True
                except Exception as exc:  # noqa: BLE001 -- recorded, reported by the caller
                    rec.error = str(exc)
                    rec.done = True
            if stop_poll.is_set() and not dirty and (
                    time.perf_counter() > stop_deadline[0] or all(r.done for r in run.timings)):
                for r in run.timings:
                    r.done = True
                return

    stop_deadline = [float("inf")]
    poll_thread = threading.Thread(target=poller, name="client-poller", daemon=True)
    if consumers and client == "poller":
        poll_thread.start()

    def consume(rec: RequestTiming, stream) -> None:
        try:
            for chunk in stream:
                now = time.perf_counter()
                if rec.first_recv is None:
                    rec.first_recv = now
                rec.last_recv = now
                rec.samples += chunk.sample_count
                rec.chunks += 1
        except Exception as exc:  # noqa: BLE001 -- recorded, reported by the caller
            rec.error = str(exc)
        rec.done = True

    with loop, ThreadPoolExecutor(max_workers=max_clients, thread_name_prefix="client") as clients:
        origin = time.perf_counter()
        for req in trace:
            _wait_until(origin + req.send_at)
            now = time.perf_counter()
            if run.window is not None and run.window[1] is not None:
                inside = [r for r in run.timings if run.window[0] <= r.send_time < run.window[1]]
                if all(r.done for r in inside) or now - run.window[1] > drain_seconds:
                    break
            rid, stream = loop.submit(req.text)
            rec = RequestTiming(rid, req.text, time.perf_counter())
            push = stream._push

            def timed_push(chunk, _push=push, _rec=rec):
                if _rec.first_push is None:
                    _rec.first_push = time.perf_counter()
                _push(chunk)

            stream._push = timed_push
            if consumers and client == "poller":
                def notify(fn, _pair=(rec, stream)):
                    def inner(*a):   # the report sink wakes the poller once per iteration
                        fn(*a)
                        dirty.append(_pair)
                    return inner
                stream._push = notify(stream._push)
                for name in ("_finish", "_fail", "_cancel"):
                    setattr(stream, name, notify(getattr(stream, name)))
            with lock:
                run.timings.append(rec)
            if consumers and client == "threads":
                clients.submit(consume, rec, stream)
            elif not consumers:  # server-side timing only
                rec.done = True
        else:  # trace exhausted before the window closed: let in-flight requests finish
            end = time.perf_counter() + tail_seconds
            while time.perf_counter() < end and not all(r.done for r in run.timings):
                time.sleep(0.001)
    if poll_thread.is_alive():
        stop_deadline[0] = time.perf_counter() + 1.0
        stop_poll.set()
        wake.set()
        poll_thread.join(timeout=5.0)
    return run


def merge_rank_stats(local: dict, dist=None) -> dict | None:
    """Multi-rank bench aggregation (one pool per GPU, no data-path collective).

    ``local`` holds this rank's per-request latency lists (``fcl``, ``fcl_c``,
    ``lcl``, ``rtf``), its timed-window length ``window`` and counters.  Rank 0
    receives the concatenated lists, the MAX window over ranks (device time of
    the slowest rank) and summed counters; other ranks get None.
    """
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return dict(local)
    world = dist.get_world_size()
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    if dist.get_rank() != 0:
        return None
    merged = {k: [x for g in gathered for x in g[k]] for k in ("fcl", "fcl_c", "lcl", "rtf")}
    merged["window"] = max(g["window"] for g in gathered)
    for k in ("missing", "launch", "h2d", "d2h"):
        merged[k] = sum(g.get(k, 0) for g in gathered)
    merged["per_rank_window"] = [g["window"] for g in gathered]
    return merged


def serve_router(router, trace: list[TimedRequest], *, warmup_seconds: float, timed_seconds: float,
                 drain_seconds: float = 5.0, tail_seconds: float = 60.0) -> ServeRun:
    """``serve`` for the multi-GPU path: plays ``trace`` against a :class:`router.Router` (one pool
    per GPU worker process).  The window is ``[warmup_seconds, warmup_seconds + timed_seconds)``
    after the first send; every request sent inside it is measured.  ``first_push`` is the
    worker-side time its first chunk became visible (CLOCK_MONOTONIC, same clock as here),
    ``first_recv`` the time this process's poller received it from the router."""
    run = ServeRun(timings=[])
    lock = threading.Lock()
    live: list = []
    stop_poll = threading.Event()

    def poller() -> None:
        pending: list = []
        while not (stop_poll.is_set() and not pending and not live):
            time.sleep(0.001)
            with lock:
                pending.extend(live)
                live.clear()
            keep = []
            for rec, stream in pending:
                try:
                    while True:
                        chunk = stream.get(timeout=0)
                        now = time.perf_counter()
                        if chunk is None:
                            rec.done = True
                            break
                        if rec.first_recv is None:
                            rec.first_recv = now
                        rec.last_recv = now
                        rec.samples += chunk.sample_count
                        rec.chunks += 1
                except queue.Empty:
                    keep.append((rec, stream))
                except Exception as exc:  # noqa: BLE001 -- recorded, reported by the caller
                    rec.error = str(exc)
                    rec.done = True
            pending = keep
            if stop_poll.is_set():   # one last pass after the stop; later chunks are not measured
                return

    th = threading.Thread(target=poller, name="router-client-poller", daemon=True)
    th.start()
    origin = time.perf_counter()
    w0, w1 = origin + warmup_seconds, origin + warmup_seconds + timed_seconds
    run.window = (w0, w1)
    for req in trace:
        _wait_until(origin + req.send_at)
        now = time.perf_counter()
        if now >= w1:
            inside = [r for r in run.timings if w0 <= r.send_time < w1]
            if all(r.done for r in inside) or now - w1 > drain_seconds:
                break
        rid, stream = router.submit(req.text)
        rec = RequestTiming(rid, req.text, time.perf_counter())
        with lock:
            run.timings.append(rec)
            live.append((rec, stream))
    else:
        end = time.perf_counter() + tail_seconds
        while time.perf_counter() < end and not all(r.done for r in run.timings):
            time.sleep(0.005)
    stop_poll.set()
    th.join(timeout=10.0)
    for rec in run.timings:
        rec.first_push = router.first_push.get(rec.request_id)
    return run


def warm_up(modules: PipelineModules, cfg, seed: int = 7, max_batch: int = 512) -> None:
    """Untimed warm-up of every serving code path before a measurement: decoder CUDA graphs of
    every batch bucket, vocoder work buffers, pinned host blocks (engine.prepare_graphs), then a
    Poisson second and bursts of simultaneous arrivals (large encoder batches, tensor maps, lazy
    module loading, allocator pools).  Also the router workers' ``WorkerSpec.warmup``."""
    engine = getattr(modules, "engine", None)
    if engine is not None and hasattr(engine, "prepare_graphs"):
        engine.prepare_graphs(max_batch=max_batch)
    lex = default_lexicon()
    serve(modules, cfg, poisson_trace(50, 1.0, seed=seed, lexicon=lex), warmup_iters=0, timed_iters=2,
          drain_seconds=0.0)
    rng = random.Random(seed + 1)
    for burst in (8, 32, 64):
        serve(modules, cfg, [TimedRequest(0.0, random_text(rng, 20, 200, lex)) for _ in range(burst)],
              warmup_iters=0, timed_iters=None, drain_seconds=0.0)
