"""Host mirror (frontend, pool, iteration loop) vs the reference's recorded behaviour.

Scheduling tables in ``tests/golden/schedules.json`` were recorded by
running the reference ``run_iteration`` (``tools/make_golden.py``); here the
same scripts run through this package's scheduler with the oracle modules
and must produce identical IterationReports (SURVEY §8c "pins on
scheduling").  Mirrors ``pkg/tests/test_scheduler.py`` semantics.
"""

import io
import json
import queue
import threading
import time

import numpy as np
import pytest

from oracle.modules import cpu_modules
from paper_2211_13939_b200.domain import ConfigError, PipelineConfig, config_from_mapping, parse_kv, validate_config
from paper_2211_13939_b200.frontend import run_frontend
from paper_2211_13939_b200.scheduler import (ChunkStream, CostModel, ModuleCost, PipelineModules,
                                             PoolClosed, RequestCancelled, RequestFailed, RequestPool,
                                             SchedulerLoop, _wait_until, latency_bounds, run_iteration,
                                             write_iteration_log)

SHORT, MEDIUM, LONG = "你们好", "欢迎收听今天新闻。", "欢迎大家收听今天下午新闻播报"


def table(reports):
    return [[list(r.frontend_ids), list(r.encoder_ids), list(r.decoder_ids), list(r.vocoder_ids),
             list(r.completed_ids), list(r.failed_ids)] for r in reports]


def drain(pool, modules, cfg, limit=2000):
    reps = []
    while pool.pending():
        reps.append(run_iteration(pool, modules, CostModel.zero(), cfg, step_index=len(reps)))
        assert len(reps) < limit
    return reps


def test_frontend_matches_reference(golden_frontend, lexicon):
    for text in golden_frontend["texts"]:
        fo = run_frontend(text, lexicon)
        want = golden_frontend["outputs"][text]
        for key, val in want.items():
            assert list(getattr(fo, key)) == val, (text, key)


def test_calibrated_fixture_lengths(texts, lexicon):
    for cls, n in (("short", 6), ("medium", 18), ("long", 30)):
        for t in texts[cls]:
            assert run_frontend(t, lexicon).seq_len == n


@pytest.mark.parametrize("ol", [4, 8])
def test_fig2_replay(golden_schedules, lexicon, ol):
    cfg = PipelineConfig(overlap_frames=ol)
    mods = cpu_modules(lexicon, cfg)
    pool, reps = RequestPool(), []

    def step():
        reps.append(run_iteration(pool, mods, CostModel.zero(), cfg, step_index=len(reps)))

    four, five = "欢迎收听新闻播报", "欢迎收听今天新闻。"
    pool.submit(four)
    step(), step()
    pool.submit(four), pool.submit(five)
    for _ in range(4):
        step()
    pool.submit(four)
    step()
    while pool.pending():
        step()
    assert table(reps) == golden_schedules[f"fig2_ol{ol}"]


@pytest.mark.parametrize("name,ol", [("random_a", 4), ("random_b", 8)])
def test_random_admission_scripts(golden_schedules, lexicon, name, ol):
    cfg = PipelineConfig(overlap_frames=ol)
    mods = cpu_modules(lexicon, cfg)
    script = golden_schedules[name]["script"]
    pool, reps = RequestPool(), []
    for batch in script:
        for text in batch:
            pool.submit(text)
        reps.append(run_iteration(pool, mods, CostModel.zero(), cfg, step_index=len(reps)))
    assert not pool.pending()
    assert table(reps) == golden_schedules[name]["table"]


def test_poisoned_item_fails_alone(golden_schedules, lexicon, cfg):
    mods = cpu_modules(lexicon, cfg)

    def fe(texts):
        if "毒" in texts:
            raise RuntimeError("poisoned batch")
        return mods.frontend_batch(texts)

    poisoned = PipelineModules(fe, mods.encoder_batch, mods.decoder_batch, mods.vocoder_batch)
    pool = RequestPool()
    streams = [pool.submit(t)[1] for t in golden_schedules["poisoned"]["texts"]]
    assert table(drain(pool, poisoned, cfg)) == golden_schedules["poisoned"]["table"]
    with pytest.raises(RequestFailed):
        streams[1].get()
    assert len(list(streams[0])) == 2


def test_admission_and_first_iteration(lexicon, cfg):
    mods = cpu_modules(lexicon, cfg)
    pool = RequestPool()
    rid, stream = pool.submit(SHORT)
    assert rid == 1 and pool.pending()
    rep = run_iteration(pool, mods, CostModel.zero(), cfg)
    assert rep.frontend_ids == rep.encoder_ids == rep.decoder_ids == rep.vocoder_ids == (rid,)
    chunk = stream.get(timeout=1.0)
    assert chunk.sample_offset == 0 and chunk.sample_count == 32 * 256 - 1024
    assert pool.items[rid].module_indicator == 1
    rep = run_iteration(pool, mods, CostModel.zero(), cfg)
    assert rep.frontend_ids == () and rep.completed_ids == (rid,)
    assert rid not in pool.items
    assert len(list(stream)) == 1 and stream.get() is None and stream.get() is None


def test_hundred_submits_join_one_iteration(lexicon, cfg):
    mods = cpu_modules(lexicon, cfg)
    pool = RequestPool()
    for _ in range(100):
        pool.submit(SHORT)
    rep = run_iteration(pool, mods, CostModel.zero(), cfg)
    assert len(rep.frontend_ids) == len(rep.decoder_ids) == 100


def test_pool_errors_and_shutdown():
    with pytest.raises(ValueError, match="empty"):
        RequestPool().submit("")
    pool = RequestPool()
    _, stream = pool.submit(SHORT)
    assert pool.shutdown() == [1]
    with pytest.raises(RequestCancelled):
        stream.get()
    with pytest.raises(PoolClosed):
        pool.submit(SHORT)
    with pytest.raises(queue.Empty):
        ChunkStream(1).get(timeout=0.01)


def test_unique_ids_under_concurrent_submits():
    pool, ids, lock = RequestPool(), [], threading.Lock()

    def worker():
        for _ in range(50):
            rid, _ = pool.submit(SHORT)
            with lock:
                ids.append(rid)

    threads = [threading.Thread(target=worker) for _ in range(8)]
    [t.start() for t in threads]
    [t.join() for t in threads]
    assert len(set(ids)) == 400


def test_cost_model_and_wait(lexicon, cfg):
    assert ModuleCost(0.004, 0.0005).duration(10) == pytest.approx(0.009)
    with pytest.raises(ValueError):
        ModuleCost(-0.001, 0.0)
    m = CostModel.from_mapping({"cost_decoder_base": "0.01"})
    assert m.decoder.base_seconds == 0.01 and m.frontend.base_seconds == 0.0
    t = time.perf_counter()
    _wait_until(t + 0.02)
    assert 0.0195 <= time.perf_counter() - t <= 0.03
    mods = cpu_modules(lexicon, cfg)
    cost = CostModel(ModuleCost(0.002), ModuleCost(0.003), ModuleCost(0.008), ModuleCost(0.005))
    pool = RequestPool()
    pool.submit(SHORT)
    rep = run_iteration(pool, mods, cost, cfg)
    assert rep.step_seconds == pytest.approx(0.018, abs=0.005)
    assert rep.charged_seconds == pytest.approx(0.018)


def test_loop_serves_and_cancels(lexicon, cfg):
    loop = SchedulerLoop(cpu_modules(lexicon, cfg), CostModel.zero(), cfg).start()
    _, stream = loop.submit(MEDIUM)
    assert len(list(stream)) == 5
    reports = loop.stop()
    assert reports and [r.step_index for r in reports] == list(range(len(reports)))
    with pytest.raises(PoolClosed):
        loop.submit(SHORT)


def test_latency_bounds_and_log(lexicon, cfg):
    assert latency_bounds(0.03, 0.01) == pytest.approx((0.01, 0.04, 0.025))
    with pytest.raises(ValueError):
        latency_bounds(-1, 0)
    pool = RequestPool()
    pool.submit(SHORT), pool.submit(MEDIUM)
    reps = drain(pool, cpu_modules(lexicon, cfg), cfg)
    sink = io.StringIO()
    write_iteration_log(reps, sink)
    parsed = [json.loads(x) for x in sink.getvalue().strip().split("\n")]
    assert parsed[0]["batch_sizes"]["frontend"] == 2 and parsed[-1]["completed"] == [2]


def test_config_validation():
    assert validate_config(PipelineConfig()) == PipelineConfig()
    with pytest.raises(ConfigError, match="overlap must be < chunk"):
        validate_config(PipelineConfig(overlap_frames=32))
    with pytest.raises(ConfigError):
        validate_config(PipelineConfig(stop_threshold=1.0))
    assert config_from_mapping(parse_kv("overlap_frames = 8  # x\n\n")).overlap_frames == 8
    with pytest.raises(ConfigError):
        parse_kv("novalue\n")


def test_step_granular_admission_preserves_chunks(lexicon, cfg):
    """The opt-in step-granular mode (run_iteration_steps): requests join the decode at the next
    8-step sub-iteration, yet every request's chunks (offsets, counts, samples) equal single-request
    synthesis exactly -- only batch composition and timing change (Tier-S oracle modules)."""
    import random

    from oracle import tier_s as orc
    from oracle.modules import cpu_modules
    from paper_2211_13939_b200.frontend import run_frontend
    from paper_2211_13939_b200.harness import random_text
    from paper_2211_13939_b200.scheduler import CostModel, RequestPool, run_iteration_steps
    rng = random.Random(12)
    texts = [random_text(rng, 2, 30, lexicon) for _ in range(12)]
    admit_at = sorted(rng.randrange(0, 40) for _ in texts)
    mods = cpu_modules(lexicon, cfg)
    pool, streams, partial, it = RequestPool(), {}, {}, 0
    joined_mid_chunk = False
    while it <= max(admit_at) or pool.pending():
        for k, t in enumerate(texts):
            if admit_at[k] == it:
                streams[k] = pool.submit(t)[1]
                joined_mid_chunk |= bool(partial)
        rep = run_iteration_steps(pool, mods, CostModel.zero(), cfg, step_index=it, sub_steps=8, partial=partial)
        assert not rep.failed_ids
        it += 1
    assert joined_mid_chunk   # some request was admitted while others were mid-chunk
    for k, t in enumerate(texts):
        fo = run_frontend(t, lexicon)
        want, _ = orc.synthesize(fo.phonemes, fo.pw, fo.pph, fo.iph)
        got = list(streams[k])
        assert [c.sample_offset for c in got] == [o for _, o in want]
        for c, (w, _) in zip(got, want):
            np.testing.assert_allclose(c.samples, w, rtol=0, atol=1e-12)
