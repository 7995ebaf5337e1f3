"""The multi-GPU serving path (C4) on real GPU modules: router + 2 worker processes, both on
cuda:0 here (one GPU per gpurun box).  Each worker's recorded admission schedule must replay
through run_iteration to the identical per-worker IterationReports, and each
request's audio must match single-request synthesis on the oracle (SNR >= 40 dB), whichever worker
served it."""

import random

import numpy as np
import pytest

from oracle import tier_r as orc
from oracle.modules import cpu_modules
from paper_2211_13939_b200.domain import PipelineConfig
from paper_2211_13939_b200.frontend import run_frontend
from paper_2211_13939_b200.harness import random_text
from paper_2211_13939_b200.router import gpu_router, wait_all
from paper_2211_13939_b200.scheduler import CostModel, RequestPool, run_iteration
from paper_2211_13939_b200.weights import tier_r_weights

pytestmark = pytest.mark.gpu


def test_router_two_gpu_workers(lexicon):
    cfg = PipelineConfig()
    rng = random.Random(31)
    texts = [random_text(rng, 8, 40, lexicon) for _ in range(10)]
    with gpu_router(2, cfg, tier="r", policy="mod", devices=["cuda:0", "cuda:0"]) as router:
        ids, streams = zip(*[router.submit(t) for t in texts])
        results = wait_all(streams, timeout=300)
    assert [router.placement[i] for i in ids] == [(i - 1) % 2 for i in ids]
    assert not router.dead
    w = tier_r_weights(0)
    for text, chunks in list(zip(texts, results))[:4]:
        fo = run_frontend(text, lexicon)
        want, _, _ = orc.synthesize(w, fo.phonemes, fo.pw, fo.pph, fo.iph)
        assert [c.sample_offset for c in chunks] == [o for _, o in want]
        snr = orc.snr_db(np.concatenate([s for s, _ in want]), np.concatenate([c.samples for c in chunks]))
        assert snr >= 40.0, snr
    # per-worker schedule replay (value-independent decisions: the stand-in modules suffice)
    by_id = dict(zip(ids, texts))
    for wk in range(2):
        pool, mods, reps, local = RequestPool(), cpu_modules(lexicon, cfg), [], {}
        for batch in router.admissions[wk]:
            for gid in batch:
                lid, _ = pool.submit(by_id[gid])
                local[lid] = gid
            reps.append(run_iteration(pool, mods, CostModel.zero(), cfg, step_index=len(reps)))
        replay = [([local[i] for i in r.decoder_ids], [local[i] for i in r.completed_ids]) for r in reps]
        recorded = [(d, c) for _, d, c in router.reports[wk]]
        assert replay == recorded[:len(replay)]
        assert all(not d for d, _ in recorded[len(replay):])
