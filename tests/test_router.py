"""Multi-GPU host router (C4) on CPU: 2 worker processes running the oracle modules.

Checks request sharding (no cross-request interaction: every request's
audio equals single-request synthesis), deterministic placement, and that
each worker's recorded admission schedule replays through run_iteration to
the identical per-worker IterationReports (SURVEY §8e parity across GPU
counts).
"""

import numpy as np
import pytest

from oracle import tier_s as orc
from oracle.modules import cpu_modules
from paper_2211_13939_b200.domain import PipelineConfig
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend
from paper_2211_13939_b200.harness import random_text
from paper_2211_13939_b200.router import Router, WorkerSpec, wait_all
from paper_2211_13939_b200.scheduler import CostModel, RequestPool, run_iteration

import random


@pytest.mark.parametrize("policy", ["mod", "least_frames"])
def test_router_two_workers(policy):
    cfg = PipelineConfig()
    lex = default_lexicon()
    rng = random.Random(5)
    texts = [random_text(rng, 2, 14, lex) for _ in range(24)]
    specs = [WorkerSpec("oracle.modules:cpu_modules", None, cfg, {}) for _ in range(2)]
    with Router(specs, policy=policy) as router:
        ids, streams = zip(*[router.submit(t) for t in texts])
        results = wait_all(streams, timeout=120)
    if policy == "mod":
        assert [router.placement[i] for i in ids] == [(i - 1) % 2 for i in ids]
    assert set(router.placement.values()) == {0, 1}
    for text, chunks in zip(texts, results):
        fo = run_frontend(text, lex)
        want, _ = orc.synthesize(fo.phonemes, fo.pw, fo.pph, fo.iph)
        assert [c.sample_offset for c in chunks] == [o for _, o in want]
        np.testing.assert_allclose(np.concatenate([c.samples for c in chunks]),
                                   np.concatenate([w for w, _ in want]), rtol=0, atol=1e-12)
    # per-worker schedule replay: same admissions -> same decoder batches and completions
    by_id = dict(zip(ids, texts))
    for w in range(2):
        admitted = [a for a in router.admissions[w]]
        pool, mods, reps, local = RequestPool(), cpu_modules(lex, cfg), [], {}
        for batch in admitted:
            for gid in batch:
                lid, _ = pool.submit(by_id[gid])
                local[lid] = gid
            reps.append(run_iteration(pool, mods, CostModel.zero(), cfg, step_index=len(reps)))
        replay = [([local[i] for i in r.decoder_ids], [local[i] for i in r.completed_ids]) for r in reps]
        recorded = [(d, c) for _, d, c in router.reports[w]]
        assert replay == recorded[:len(replay)]
        assert all(not d for d, _ in recorded[len(replay):])


def test_dead_worker_fails_its_streams():
    """A worker process that dies mid-stream: its open streams fail (no hang), the other
    worker's requests still complete."""
    from paper_2211_13939_b200.scheduler import RequestFailed
    cfg, lex = PipelineConfig(), default_lexicon()
    specs = [WorkerSpec("oracle.modules:cpu_modules", None, cfg),
             WorkerSpec("oracle.modules:crashing_modules", None, cfg)]
    rng = random.Random(9)
    short = [random_text(rng, 2, 6, lex) for _ in range(4)]
    long_text = random_text(rng, 40, 40, lex)
    with Router(specs, policy="mod") as router:
        streams = [router.submit(t)[1] for t in short[:3]] + [router.submit(long_text)[1]]  # ids 1..4
        ok = []
        for i, s in enumerate(streams):
            try:
                ok.append(len(wait_all([s], timeout=60)[0]) > 0)
            except RequestFailed as exc:
                assert "died" in str(exc)
                ok.append(False)
    assert router.dead == [1]
    assert ok[0] and ok[2]            # worker 0 (ids 1, 3) unaffected
    assert not ok[3]                  # the crash request (id 4 -> worker 1) failed, no hang
