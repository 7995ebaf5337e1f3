"""Serving benchmark: first-chunk latency (FCL) p50/p99 under Poisson load (BASELINE config C3)
and max QPS at p99 FCL < 80 ms.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--qps Q] [--impl ours|reference]

Workload (``config.workload``): Poisson arrivals at ``--qps`` per GPU (default 100, weak
scaling), texts of U{20..200} characters drawn from the bundled lexicon's single-character
entries (seeded), random-init Tacotron2 (512 enc, 1024 LSTM) + HiFi-GAN V1 at 22.05 kHz, chunk 32
frames, overlap 4, through this package's request pool + module-wise dynamic batching loop and
its GPU modules (``build_modules(..., tier="r")``).

A "step" is ONE SECOND of Poisson serving: after W warm-up steps (seconds of load) exactly K
steps are timed (K seconds, ~100 K requests at 100 QPS) and every request sent inside that window
is measured:

* ``value``  p99 FCL in ms at the server boundary: submit() to the first AudioChunk becoming
  visible on the request's ChunkStream.
* ``e2e``    the same p99 measured by a client thread receiving the chunk through the public
  ``SchedulerLoop.submit`` / ``ChunkStream`` API (text in, host float32 audio out; the H2D of
  tokens / plans and the D2H of audio are inside).

N = 1 serves in-process (one pool, one GPU).  N > 1 (torchrun, one rank per GPU) serves through
``router.Router``: rank 0 runs the router and one worker process per GPU (own CUDA context,
weights, pool and loop; no collectives), the other ranks only wait on a host barrier.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "first-chunk latency p50/p99 (ms) and max QPS at <80ms p99, 1/2/4/8 B200"
SLO_MS = 80.0


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return {**json.loads(p.read_text()), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed window."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus: str):
        self.gpus, self.proc = gpus, None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpus, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


_T0 = time.perf_counter()


def log(msg: str) -> None:
    """Progress on stderr (the JSON line is the only stdout output)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def _pct(values, p):
    from paper_2211_13939_b200.harness import nearest_rank
    return nearest_rank(values, p) if values else None


def _cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def _window_stats(run, end_pad: float = 2.0) -> dict:
    """Latencies of the requests sent inside run.window; a request without a first chunk counts
    as censored at the window end + end_pad."""
    t0, t1 = run.window
    inside = [r for r in run.timings if t0 <= r.send_time < t1]
    cens = t1 + end_pad
    fcl = [1e3 * (r.fcl if r.fcl is not None else cens - r.send_time) for r in inside]
    fcl_c = [1e3 * r.fcl_client for r in inside if r.fcl_client is not None]
    seg = []   # stationarity: p99 per third of the window
    for k in range(3):
        a, b = t0 + k * (t1 - t0) / 3, t0 + (k + 1) * (t1 - t0) / 3
        part = [1e3 * r.fcl for r in inside if a <= r.send_time < b and r.fcl is not None]
        seg.append(round(_pct(part, 99), 3) if part else None)
    return {"requests": len(inside), "p50": _pct(fcl, 50), "p99": _pct(fcl, 99),
            "c50": _pct(fcl_c, 50), "c99": _pct(fcl_c, 99),
            "censored": sum(1 for r in inside if r.fcl is None),
            "failed": sum(1 for r in inside if r.error is not None and "cancelled" not in r.error),
            "p99_by_third": seg, "window_s": t1 - t0,
            "lcl": [1e3 * r.lcl for r in inside if r.lcl is not None and r.error is None],
            "rtf": [r.lcl / (r.samples / 22050.0) for r in inside if r.lcl is not None and r.error is None and r.samples]}


# ------------------------------------------------------------------ CPU baselines (test infrastructure)
def cpu_port_baseline(seconds: float, seed: int) -> dict:
    """The oracle Tier-R CPU implementation (torch-CPU fp32 Tacotron2 + HiFi-GAN V1, all host
    threads) behind the same scheduler: (a) first-chunk latency of ONE 50-char request on an idle
    pool (the floor of its p99 FCL at any load, so max QPS at p99 < 80 ms is 0 when it exceeds 80
    ms), (b) saturated throughput -- audio chunks per second with 32 ragged requests pooled --
    over a bounded sample of `seconds`."""
    import torch

    from oracle.modules import cpu_modules_r
    from paper_2211_13939_b200.domain import PipelineConfig
    from paper_2211_13939_b200.frontend import default_lexicon
    from paper_2211_13939_b200.harness import random_text
    from paper_2211_13939_b200.scheduler import CostModel, RequestPool, run_iteration
    from paper_2211_13939_b200.weights import tier_r_weights

    cores = _cores()
    torch.set_num_threads(cores)
    cfg, lex = PipelineConfig(), default_lexicon()
    w = tier_r_weights(0)
    mods = cpu_modules_r(lex, cfg, w)
    rng = random.Random(seed + 999)
    fcl = []
    for _ in range(3):   # idle-pool FCL of a 50-char request (first one warms the allocator)
        pool = RequestPool()
        t0 = time.perf_counter()
        _, st = pool.submit(random_text(rng, 50, 50, lex))
        run_iteration(pool, mods, CostModel.zero(), cfg)
        st.get(timeout=0)
        fcl.append(1e3 * (time.perf_counter() - t0))
    pool, chunks, it = RequestPool(), 0, 0
    for _ in range(32):
        pool.submit(random_text(rng, 20, 200, lex))
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds and pool.pending():
        rep = run_iteration(pool, mods, CostModel.zero(), cfg, step_index=it)
        chunks += len(rep.vocoder_ids)
        it += 1
    dt = time.perf_counter() - t0
    single = sorted(fcl[1:])[0]
    cps = chunks / dt
    # a U{20..200}-char request is ~57 chunks on average: above cps / 57 requests per
    # second the CPU falls behind the arrivals and its queue (and FCL) grows without bound
    qps_bound = 0.0 if single > SLO_MS else cps / 57.0
    return {"value": round(single, 1), "unit": "ms", "cores": cores, "kind": "port",
            "single_request_fcl_ms": round(single, 1), "max_qps_p99_under_80ms_upper_bound": round(qps_bound, 3),
            "chunks_per_s_saturated": round(cps, 2), "iterations": it,
            "sample": f"oracle Tier-R CPU modules (torch fp32, {cores} threads) behind the same scheduler: idle-pool "
                      f"FCL of one 50-char request, then {dt:.0f} s of 32 pooled U{{20..200}}-char requests "
                      "(saturated chunks/s)"}


def reference_standin_baseline(qps_levels, seconds: float, seed: int) -> dict | None:
    """The reference's OWN stock path, unmodified, from baseline/_ref: ``SchedulerLoop(
    build_modules(default_lexicon(), PipelineConfig()), CostModel.zero(), cfg)`` (reference
    scheduler.py:266,548) -- its deterministic stand-in networks, not
    Tacotron2 / HiFi-GAN -- on the same Poisson U{20..200} workload: p99 FCL per QPS level and the
    max QPS with p99 < 80 ms.  One GIL-bound loop thread."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "incrtts" / "scheduler.py").exists():
        return None
    sys.path.insert(0, str(ref))
    try:
        import incrtts
        from incrtts.scheduler import CostModel, SchedulerLoop, build_modules
    finally:
        sys.path.remove(str(ref))
    from paper_2211_13939_b200.frontend import default_lexicon
    from paper_2211_13939_b200.harness import poisson_trace
    lex = incrtts.default_lexicon() if hasattr(incrtts, "default_lexicon") else None
    cfg = incrtts.PipelineConfig()
    rows = []
    for q in qps_levels:
        trace = poisson_trace(q, seconds, seed=seed + 77, lexicon=default_lexicon())
        sent, first = {}, {}
        with SchedulerLoop(build_modules(lex, cfg), CostModel.zero(), cfg) as loop:
            origin = time.perf_counter()
            for r in trace:
                while time.perf_counter() < origin + r.send_at:
                    time.sleep(0.0005)
                rid, stream = loop.submit(r.text)
                sent[rid] = time.perf_counter()
                push = stream._push
                stream._push = (lambda c, _p=push, _r=rid: (first.setdefault(_r, time.perf_counter()), _p(c)))
            end = time.perf_counter() + 2.0
            while len(first) < len(sent) and time.perf_counter() < end:
                time.sleep(0.01)
            stop = time.perf_counter()
        fcl = [1e3 * (first.get(r, stop) - t) for r, t in sent.items()]
        rows.append({"qps": q, "p50_ms": round(_pct(fcl, 50), 2), "p99_ms": round(_pct(fcl, 99), 2),
                     "requests": len(fcl), "censored": len(sent) - len(first)})
        log(f"reference stand-in {q:g} QPS: p99 {rows[-1]['p99_ms']} ms")
        if rows[-1]["p99_ms"] > SLO_MS:
            break
    ok = [r["qps"] for r in rows if r["p99_ms"] < SLO_MS]
    return {"path": "reference incrtts SchedulerLoop + build_modules (stand-in arithmetic), baseline/_ref",
            "rows": rows, "max_qps_p99_under_80ms": max(ok) if ok else 0.0, "cores": 1,
            "window_s": seconds}


def run_reference(args) -> None:
    """Reference arm (driver: --impl reference): the CPU implementation of the same Tier-R path on
    the box's host cores -- the oracle port, as the reference has no networks -- on a bounded
    sample of this arm's workload, plus the reference's own stand-in path.  Rank 0 only."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    t0 = time.perf_counter()
    res = cpu_port_baseline(args.cpu_seconds, args.seed)
    ref = reference_standin_baseline([2.0, 4.0, 8.0, 12.0, 16.0, 24.0, 32.0], 10.0, args.seed)
    wall = time.perf_counter() - t0
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * wall / max(args.steps, 1), 3),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"C3 workload, CPU port: a single 50-char request on an idle pool (the p99 FCL "
                                   f"floor at any QPS) + saturated chunks/s; Tacotron2+HiFi-GAN V1 random init",
                       "qps_per_gpu": args.qps},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "max_qps_p99_under_80ms_upper_bound": res["max_qps_p99_under_80ms_upper_bound"],
            "chunks_per_s_saturated": res["chunks_per_s_saturated"],
            "reference_standin": ref,
            "e2e": {"value": res["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def _flush_wrapped(mods, engine, device):
    """Every decoder call starts after a 256 MB write on the engine stream (> 126 MB L2): the
    weights are re-read from HBM each iteration (timing rule: flush L2 between timed steps)."""
    import torch

    from paper_2211_13939_b200.scheduler import PipelineModules
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    dec_fn = mods.decoder_batch

    def decoder_with_flush(pairs):
        with torch.cuda.stream(engine.stream):
            flush.fill_(1)
        return dec_fn(pairs)

    out = PipelineModules(mods.frontend_batch, mods.encoder_batch, decoder_with_flush, mods.vocoder_batch)
    for k in ("engine", "frontend_prefetch", "decoder_steps", "concat_mels"):
        if hasattr(mods, k):
            object.__setattr__(out, k, getattr(mods, k))
    return out


def run_single(args) -> dict:
    """N = 1: one pool + loop in this process."""
    import torch

    from paper_2211_13939_b200.domain import PipelineConfig
    from paper_2211_13939_b200.frontend import default_lexicon
    from paper_2211_13939_b200.harness import poisson_trace, serve, warm_up
    from paper_2211_13939_b200.modules import build_modules

    torch.cuda.set_device(0)
    cfg, lex = PipelineConfig(), default_lexicon()
    mods = build_modules(lex, cfg, tier="r", device="cuda:0")
    engine = mods.engine
    if args.precision:
        engine.set_precision(args.precision)
    log("engine built")
    warm_up(mods, cfg, seed=args.seed + 7)
    log("warm-up done (graphs captured)")
    if args.l2_flush:
        mods = _flush_wrapped(mods, engine, "cuda:0")
    torch.cuda.synchronize()
    peaks = _peaks()
    sampler = ClockSampler("0")
    marks = {}

    def on_window(kind, idx):
        torch.cuda.synchronize()
        if kind == "start":
            engine.timers = []
            marks["start"] = (engine.launches, engine.h2d_bytes, engine.d2h_bytes, time.perf_counter())
            sampler.start()
        else:
            marks["clocks"] = sampler.stop()
            marks["end"] = (engine.launches, engine.h2d_bytes, engine.d2h_bytes, time.perf_counter())
            marks["timers"], engine.timers = engine.timers, None

    trace = poisson_trace(args.qps, 3600.0, seed=args.seed + 1000, lexicon=lex)
    log(f"C3 main window: {args.qps:g} QPS, {args.steps} s timed after {args.warmup} s")
    run = serve(mods, cfg, trace, warmup_iters=3, warmup_seconds=float(args.warmup), timed_iters=None,
                timed_seconds=float(args.steps), on_window=on_window, drain_seconds=args.drain_seconds)
    torch.cuda.synchronize()
    st = _window_stats(run)
    t0, t1 = run.window
    batch = [len(rep.decoder_ids) for rep, e in zip(run.reports, run.iteration_end) if t0 < e <= t1]
    agg = {}
    for kind, e0, e1, units in marks.get("timers") or []:
        a = agg.setdefault(kind, [0.0, 0.0, 0])
        a[0] += e0.elapsed_time(e1)
        a[1] += units
        a[2] += 1
    n_steps = max(args.steps, 1)
    out = {"stats": st, "batch": batch, "agg": agg, "marks": marks, "peaks": peaks, "iterations": len(batch)}
    log(f"C3 done: p50 {st['p50']:.2f} p99 {st['p99']:.2f} ms over {st['requests']} requests")
    if args.side_configs:
        out["side_configs"] = side_configs(mods, cfg, lex, args)
    if args.sweep:
        def serve_at(q, secs):
            # module CUDA events over the whole run: each level's roofline fractions (the decoder's
            # achieved bytes/s grow with the pooled batch; the 100 QPS headline is its small-B point)
            engine.timers = []
            run = serve(mods, cfg, poisson_trace(q, 3600.0, seed=args.seed + int(q), lexicon=lex), warmup_iters=3,
                        warmup_seconds=3.0, timed_iters=None, timed_seconds=secs, drain_seconds=2.0)
            torch.cuda.synchronize()
            agg_q = {}
            for kind, e0, e1, units in engine.timers:
                a_ = agg_q.setdefault(kind, [0.0, 0.0])
                a_[0] += e0.elapsed_time(e1)
                a_[1] += units
            engine.timers = None
            dec_q, voc_q = agg_q.get("decoder"), agg_q.get("vocoder")
            run.roofline = {
                "decoder_frac_hbm": round(dec_q[1] / (dec_q[0] * 1e-3) / 1e9 / peaks["hbm_gbs"], 4) if dec_q else None,
                "vocoder_frac_bf16": (round(voc_q[1] / (voc_q[0] * 1e-3) / 1e12 / peaks["bf16_tflops_sustained"], 4)
                                      if voc_q else None)}
            return run
        out["sweep"] = qps_sweep(serve_at, [float(x) for x in args.sweep.split(",") if x], args.sweep_seconds,
                                 args.qps, st["p99"])
    out["n_steps"] = n_steps
    out["engine"] = engine
    return out


def run_multi(args, world: int) -> dict:
    """N > 1: the router + one worker process per GPU (cuda:0..N-1); called on rank 0."""
    from paper_2211_13939_b200.domain import PipelineConfig
    from paper_2211_13939_b200.frontend import default_lexicon
    from paper_2211_13939_b200.harness import poisson_trace, serve_router
    from paper_2211_13939_b200.router import gpu_router

    cfg, lex = PipelineConfig(), default_lexicon()
    log(f"starting router with {world} GPU workers")
    devices = args.router_devices.split(",") if args.router_devices else [f"cuda:{i}" for i in range(world)]
    router = gpu_router(world, cfg, tier="r", warmup="paper_2211_13939_b200.harness:warm_up", devices=devices)
    log("workers ready")
    sampler = ClockSampler(",".join(sorted({d.split(":")[-1] for d in devices})))
    try:
        qps = args.qps * world
        sampler.start()
        run = serve_router(router, poisson_trace(qps, 3600.0, seed=args.seed + 1000, lexicon=lex),
                           warmup_seconds=float(args.warmup), timed_seconds=float(args.steps),
                           drain_seconds=args.drain_seconds)
        clocks = sampler.stop()
        st = _window_stats(run)
        log(f"C4 main window: {qps:g} QPS over {world} GPUs: p99 {st['p99']:.2f} ms")
        out = {"stats": st, "clocks": clocks, "n_steps": max(args.steps, 1)}
        if args.sweep:
            out["sweep"] = qps_sweep(lambda q, secs: serve_router(
                router, poisson_trace(q, 3600.0, seed=args.seed + int(q), lexicon=lex), warmup_seconds=3.0,
                timed_seconds=secs, drain_seconds=2.0),
                [world * float(x) for x in args.sweep.split(",") if x], args.sweep_seconds, qps, st["p99"])
    finally:
        router.close()
    out["dead_workers"] = router.dead
    return out


def run_ours(args) -> None:
    world, rank, _ = _dist()
    dist = None
    if world > 1:
        import torch.distributed as dist
        # host-only rendezvous (no collectives on the data path): gloo, CPU
        dist.init_process_group("gloo")
        if rank != 0:   # rank 0 drives the router and its one-process-per-GPU workers
            dist.barrier()
            dist.destroy_process_group()
            return
    res = run_single(args) if world == 1 else run_multi(args, world)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    st = res["stats"]
    peaks = _peaks()
    line = {
        "metric": METRIC, "value": round(st["p99"], 3) if st["p99"] is not None else None, "unit": "ms",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * st["window_s"] / max(args.steps, 1), 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": res.get("dtype", "bf16"), "data": "synthetic",
        "config": {"workload": f"C3: Poisson {args.qps:g} QPS per GPU, U{{20..200}} chars (seeded, bundled lexicon), "
                               "random-init Tacotron2 (512 enc, 1024 LSTM) + HiFi-GAN V1 22.05 kHz, chunk 32, "
                               "overlap 4, tier r",
                   "step": "1 s of Poisson serving (K steps = K seconds timed)",
                   "qps_per_gpu": args.qps, "qps_total": args.qps * world,
                   "parallelism": "in-process pool" if world == 1 else f"router + {world} worker processes (pool per GPU)",
                   "l2": ("flushed: a 256 MB write on the engine stream before every iteration's decoder call "
                          "(inside the timed region)") if args.l2_flush and world == 1 else "not flushed",
                   "gc": "default CPython GC (no freeze / threshold tuning)",
                   "requests_measured": st["requests"], "requests_censored": st["censored"],
                   "requests_failed": st["failed"]},
        "p50_ms": round(st["p50"], 3) if st["p50"] is not None else None,
        "p99_ms_by_third_of_window": st["p99_by_third"],
        "lcl_p50_ms": _pct(st["lcl"], 50), "lcl_p99_ms": _pct(st["lcl"], 99),
        "rtf_mean": (sum(st["rtf"]) / len(st["rtf"])) if st["rtf"] else None,
    }
    if world == 1:
        eng, agg, marks, batch, n = res["engine"], res["agg"], res["marks"], res["batch"], res["n_steps"]
        if getattr(eng, "precision", "bf16") == "parity":
            line["dtype"] = "fp32 decoder (bf16x3-split tcgen05 gate products, fp32 accumulate); bf16 vocoder"
        else:
            line["dtype"] = "bf16"
        line["precision"] = eng.precision_label() if hasattr(eng, "precision_label") else "bf16"
        line["iterations_in_window"] = res["iterations"]
        line["pooled_batch_mean"] = round(sum(batch) / max(len(batch), 1), 1)
        line["pooled_batch_max"] = max(batch) if batch else 0
        half = len(batch) // 2
        line["pooled_batch_mean_by_half"] = [round(sum(batch[:half]) / max(half, 1), 1),
                                             round(sum(batch[half:]) / max(len(batch) - half, 1), 1)]
        iters = max(res["iterations"], 1)
        line["module_device_ms_per_iteration"] = {k: round(v[0] / iters, 3) for k, v in agg.items()}
        voc, dec = agg.get("vocoder", [0.0, 0.0, 0]), agg.get("decoder", [0.0, 0.0, 0])
        voc_tflops = voc[1] / (voc[0] * 1e-3) / 1e12 if voc[0] else None
        dec_gbs = dec[1] / (dec[0] * 1e-3) / 1e9 if dec[0] else None
        traffic = {}
        tf = ROOT / "profiles" / "ncu_traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text())
        line["roofline"] = {
            "kernel": "k_dec_persist (32-step Tacotron2 decoder chunk, one launch per iteration)", "bound": "hbm",
            "achieved": round(dec_gbs, 1) if dec_gbs else None, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(dec_gbs / peaks["hbm_gbs"], 4) if dec_gbs else None,
            "traffic": traffic.get("k_dec_persist_dram_bytes_per_launch"),
            "peak_source": peaks["source"] + " copy bandwidth",
            "algorithmic": "per step: gate + GEMV weights (36.7 MB: bf16, also in the parity mode, whose bf16-grid "
                           "weights need no low parts; 73 MB for off-grid weights) + per item 20 KB state + L x 2.5 KB "
                           "memory/processed memory; achieved = those bytes / CUDA-event time of the decoder call on "
                           "the engine stream",
            "traffic_note": traffic.get("note")}
        line["roofline_vocoder"] = {
            "kernel": "HiFi-GAN V1 chunk vocoder (k_resblock_tc fused MRF layers + k_conv_tc)", "bound": "tensor",
            "achieved": round(voc_tflops, 2) if voc_tflops else None, "peak": peaks["bf16_tflops_sustained"],
            "unit": "TFLOP/s", "frac": round(voc_tflops / peaks["bf16_tflops_sustained"], 4) if voc_tflops else None,
            "traffic": traffic.get("k_resblock_tc_dram_bytes_per_launch"),
            "peak_source": peaks["source"] + " sustained bf16", "algorithmic": "2 x 307,052,544 MAC per spliced mel frame"}
        line["e2e"] = {"value": round(st["c99"], 3) if st["c99"] is not None else None, "p50": st["c50"], "unit": "ms",
                       "h2d_bytes_per_step": int((marks["end"][1] - marks["start"][1]) / n),
                       "d2h_bytes_per_step": int((marks["end"][2] - marks["start"][2]) / n)}
        line["gpu_launches"] = int(marks["end"][0] - marks["start"][0])
        line["clocks"] = marks.get("clocks")
        if "side_configs" in res:
            line["side_configs"] = res["side_configs"]
    else:
        line["e2e"] = {"value": round(st["c99"], 3) if st["c99"] is not None else None, "p50": st["c50"], "unit": "ms",
                       "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                       "note": "client thread of the router process; H2D / D2H happen in the worker processes"}
        line["clocks"] = res["clocks"]
        line["dead_workers"] = res["dead_workers"]
    if "sweep" in res:
        line["qps_sweep"] = res["sweep"]["rows"]
        line["max_qps_p99_under_80ms"] = res["sweep"]["max_qps"]
    if not args.no_cpu_baseline:
        log("cpu baselines")
        line["cpu_baseline"] = cpu_port_baseline(args.cpu_seconds, args.seed)
        line["reference_standin"] = reference_standin_baseline([2.0, 4.0, 8.0, 12.0, 16.0, 24.0, 32.0], 10.0, args.seed)
    log("done")
    print(json.dumps(line), flush=True)


def side_configs(mods, cfg, lex, args) -> dict:
    """BASELINE configs C1 (one ~50-char request, batch 1), C2 (16 concurrent U{20..200}-char
    requests) and C5 (1000-char paragraphs every 2 s mixed with U{20..50} background)."""
    from paper_2211_13939_b200.harness import TimedRequest, poisson_trace, random_text, serve
    out = {}
    rng = random.Random(args.seed + 11)
    fcl = []
    for _ in range(10):
        run = serve(mods, cfg, [TimedRequest(0.0, random_text(rng, 50, 50, lex))], warmup_iters=0,
                    timed_iters=None, drain_seconds=0.0)
        fcl.append(1e3 * run.timings[0].fcl)
    out["c1_single_50char_fcl_ms"] = {"median": sorted(fcl)[len(fcl) // 2], "max": max(fcl), "runs": len(fcl)}
    log("C1 done")
    texts = [random_text(rng, 20, 200, lex) for _ in range(16)]
    run = serve(mods, cfg, [TimedRequest(0.0, t) for t in texts], warmup_iters=0, timed_iters=None, drain_seconds=0.0)
    out["c2_16_concurrent"] = {"fcl_max_ms": max(1e3 * r.fcl for r in run.timings),
                               "lcl_max_ms": max(1e3 * r.lcl for r in run.timings), "iterations": len(run.reports)}
    bg = poisson_trace(args.c5_qps, 25.0, lo=20, hi=50, seed=args.seed + 5, lexicon=lex)
    longs = [TimedRequest(2.0 * i + 0.5, random_text(rng, 1000, 1000, lex), "long") for i in range(12)]
    run = serve(mods, cfg, sorted(bg + longs, key=lambda r: r.send_at), warmup_iters=3, warmup_seconds=1.0,
                timed_iters=None, timed_seconds=20.0, drain_seconds=1.0)
    t0, t1 = run.window
    ins = [r for r in run.timings if t0 <= r.send_time < t1 and r.fcl is not None]
    lf = [1e3 * r.fcl for r in ins if len(r.text) >= 1000]
    sf = [1e3 * r.fcl for r in ins if len(r.text) < 1000]
    out["c5_long_paragraph_mix"] = {"background_qps": args.c5_qps, "long_requests": len(lf),
                                    "long_fcl_p50_ms": _pct(lf, 50), "long_fcl_max_ms": max(lf) if lf else None,
                                    "short_fcl_p99_ms": _pct(sf, 99), "short_requests": len(sf)}
    log("C5 done")
    out["incr_vs_non_incr"] = incr_vs_non_incr(mods, cfg, lex, args)
    log("INCR vs Non-INCR done")
    if hasattr(mods, "decoder_steps"):
        out["step_admission"] = step_admission_compare(mods, cfg, lex, args)
        log("step-granular admission done")
    eng = getattr(mods, "engine", None)
    if eng is not None and hasattr(eng, "set_precision"):
        out["precision_modes"] = precision_compare(mods, cfg, lex, args)
        log("precision modes done")
    return out


def precision_compare(mods, cfg, lex, args) -> dict:
    """north_star: "any bf16 mode reported separately" -- the same 100 QPS Poisson trace with the
    parity arithmetic (the headline) and with single bf16 gate products, 10 s windows each, plus
    each mode's decoder device time per iteration."""
    from paper_2211_13939_b200.harness import poisson_trace, serve
    eng = mods.engine
    out, mode0 = {}, eng.precision
    try:
        for mode in ("parity", "bf16"):
            eng.set_precision(mode)
            eng.prepare_graphs(max_batch=512)
            eng.timers = []
            run = serve(mods, cfg, poisson_trace(args.qps, 3600.0, seed=args.seed + 66, lexicon=lex), warmup_iters=3,
                        warmup_seconds=2.0, timed_iters=None, timed_seconds=10.0, drain_seconds=2.0)
            import torch
            torch.cuda.synchronize()
            dec = [e0.elapsed_time(e1) for kind, e0, e1, _ in eng.timers if kind == "decoder"]
            eng.timers = None
            st = _window_stats(run)
            out[mode] = {"p50_ms": st["p50"], "p99_ms": st["p99"], "requests": st["requests"], "failed": st["failed"],
                         "decoder_ms_per_call": round(sum(dec) / max(len(dec), 1), 3),
                         "label": eng.precision_label()}
    finally:
        eng.set_precision(mode0)
        eng.prepare_graphs(max_batch=512)
    return out


def step_admission_compare(mods, cfg, lex, args) -> dict:
    """North_star's "admits new requests at every decoder step" (opt-in, reported separately): the
    same Poisson trace with per-iteration admission (the reference's parity mode) and with
    step-granular admission."""
    from paper_2211_13939_b200.harness import poisson_trace, serve
    out = {"sub_steps": 8}
    for mode in ("iteration", "step"):
        run = serve(mods, cfg, poisson_trace(args.qps, 3600.0, seed=args.seed + 55, lexicon=lex), warmup_iters=3,
                    warmup_seconds=2.0, timed_iters=None, timed_seconds=10.0, drain_seconds=2.0, admission=mode)
        st = _window_stats(run)
        out[mode] = {"p50_ms": st["p50"], "p99_ms": st["p99"], "requests": st["requests"], "failed": st["failed"]}
    return out


def incr_vs_non_incr(mods, cfg, lex, args) -> dict:
    """Paper Table 1 comparison on the GPU: the same Poisson trace (U{20..200} chars) through the
    incremental pool (first-chunk latency) and through the round-based non-incremental twin
    (``baseline.py``; its only chunk is the whole waveform, so first-chunk = last-chunk latency)."""
    from paper_2211_13939_b200.baseline import BaselineServer
    from paper_2211_13939_b200.harness import poisson_trace, serve
    from paper_2211_13939_b200.scheduler import CostModel
    qps, secs = args.twin_qps, 8.0
    trace = poisson_trace(qps, secs, seed=args.seed + 21, lexicon=lex)
    run = serve(mods, cfg, trace, warmup_iters=0, timed_iters=None, drain_seconds=0.0, tail_seconds=30.0)
    incr = [1e3 * r.fcl for r in run.timings if r.fcl is not None]
    pushed, sent = {}, {}
    with BaselineServer(mods, CostModel.zero(), cfg) as srv:
        origin = time.perf_counter()
        for req in trace:
            while time.perf_counter() < origin + req.send_at:
                time.sleep(0.0005)
            rid, stream = srv.submit(req.text)
            sent[rid] = time.perf_counter()
            push = stream._push
            stream._push = (lambda c, _p=push, _r=rid: (pushed.setdefault(_r, time.perf_counter()), _p(c)))
        deadline = time.perf_counter() + 60.0
        while len(pushed) < len(sent) and time.perf_counter() < deadline:
            time.sleep(0.01)
    lat = [1e3 * (pushed[r] - t) for r, t in sent.items() if r in pushed]
    return {"qps": qps, "requests": len(trace), "incr_fcl_p50_ms": _pct(incr, 50), "incr_fcl_p99_ms": _pct(incr, 99),
            "non_incr_latency_p50_ms": _pct(lat, 50), "non_incr_latency_p99_ms": _pct(lat, 99),
            "note": "server-side: submit -> the (single, whole-waveform) chunk visible on the stream"}


def qps_sweep(serve_at, levels, seconds: float, base_qps: float, base_p99: float | None) -> dict:
    """Max QPS at p99 FCL < 80 ms: windows of `seconds` (3 s warm-up each) at increasing levels until
    one misses the SLO, then up to two bisection steps between the last pass and the first miss.
    Requests with no first chunk 2 s after the window count as censored at that time."""
    rows = []

    def level(q):
        run = serve_at(q, seconds)
        st = _window_stats(run)
        row = {"qps": q, "p50_ms": st["p50"], "p99_ms": st["p99"], "requests": st["requests"],
               "censored": st["censored"], "failed": st["failed"], "p99_ms_by_third_of_window": st["p99_by_third"],
               "window_s": round(st["window_s"], 2)}
        if getattr(run, "roofline", None):
            row["roofline"] = run.roofline
        if hasattr(run, "reports") and run.reports:
            t0, t1 = run.window
            win = [len(r.decoder_ids) for r, e in zip(run.reports, run.iteration_end) if t0 < e <= t1]
            row["pooled_batch_mean"] = round(sum(win) / max(len(win), 1), 1)
            row["ms_per_iteration"] = round(1e3 * (t1 - t0) / max(len(win), 1), 3)
        rows.append(row)
        log(f"sweep {q:g} QPS: p50 {st['p50']} p99 {st['p99']} ({st['requests']} requests)")
        return st["p99"] is not None and st["p99"] < SLO_MS and st["failed"] == 0

    last_ok, first_bad = (base_qps if base_p99 is not None and base_p99 < SLO_MS else None), None
    for q in levels:
        if level(q):
            last_ok = q
        else:
            first_bad = q
            break
    for _ in range(2):   # two bisection steps between the last pass and the first miss
        if last_ok is None or first_bad is None or first_bad - last_ok <= 20:
            break
        mid = round((last_ok + first_bad) / 2 / 5) * 5
        if level(mid):
            last_ok = mid
        else:
            first_bad = mid
    return {"rows": rows, "max_qps": last_ok}


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30, help="timed steps = seconds of Poisson serving")
    ap.add_argument("--warmup", type=int, default=5, help="warm-up steps = seconds of load before the window")
    ap.add_argument("--drain-seconds", type=float, default=10.0)
    ap.add_argument("--qps", type=float, default=100.0)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--precision", default=None, help="decoder arithmetic: parity (bf16x3 split) or bf16")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", default="200,275,350,425",
                    help="QPS levels per GPU for max QPS at p99 < 80 ms (empty: off); stops at the first miss, "
                         "then up to two bisection steps")
    ap.add_argument("--sweep-seconds", type=float, default=30.0)
    ap.add_argument("--side-configs", type=int, default=1, help="also run C1, C2, C5, INCR vs Non-INCR (1 = on)")
    ap.add_argument("--c5-qps", type=float, default=50.0)
    ap.add_argument("--twin-qps", type=float, default=30.0, help="QPS of the INCR vs Non-INCR comparison")
    ap.add_argument("--router-devices", default="",
                    help="N > 1: comma-separated worker devices (default cuda:0..N-1; e.g. cuda:0,cuda:0 to test "
                         "the router path on one GPU)")
    ap.add_argument("--l2-flush", type=int, default=1,
                    help="1: write a 256 MB buffer on the engine stream before every decoder call, so each "
                         "serving iteration starts with a cold L2 (timing rule); 0: steady-state caches")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    random.seed(args.seed)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
