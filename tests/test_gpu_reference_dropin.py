"""Drop-in proof: the REFERENCE's own scheduler -- ``incrtts.scheduler``
``RequestPool`` / ``run_iteration`` / ``SchedulerLoop`` (``pkg/src/incrtts/scheduler.py:133-188,
378-505, 548-597``), unmodified, from the installed copy in ``baseline/_ref`` -- driving this
package's Tier-R GPU modules through its ``PipelineModules`` plugin boundary.

Its IterationReports must equal the ones this package's host mirror produces over the same GPU
modules for the same admission script, and the audio must be identical bit for bit (same
batches, same kernels).  Skipped when the reference is not installed (``baseline/_ref`` is
git-ignored; it travels to the GPU box with the working tree).
"""

import random
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2211_13939_b200.domain import PipelineConfig
from paper_2211_13939_b200.harness import random_text
from paper_2211_13939_b200.scheduler import CostModel, RequestPool, run_iteration

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref_scheduler():
    if not (REF / "incrtts" / "scheduler.py").exists():
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, str(REF))
    try:
        import incrtts.scheduler as rs
    finally:
        sys.path.remove(str(REF))
    return rs


def _script(lexicon):
    rng = random.Random(77)
    texts = [random_text(rng, 10, 80, lexicon) for _ in range(7)]
    return texts, [0, 0, 1, 3, 3, 6, 9]


def _drive(pool_cls, run, cost, mods, cfg, texts, admit_at):
    pool, streams, reports, it = pool_cls(), {}, [], 0
    while it <= max(admit_at) or pool.pending():
        for k, t in enumerate(texts):
            if admit_at[k] == it:
                streams[k] = pool.submit(t)[1]
        rep = run(pool, mods, cost, cfg, step_index=it)
        reports.append((rep.frontend_ids, rep.encoder_ids, rep.decoder_ids, rep.vocoder_ids,
                        rep.completed_ids, rep.failed_ids))
        it += 1
    audio = [[(c.sample_offset, np.asarray(c.samples).copy()) for c in streams[k]] for k in range(len(texts))]
    return reports, audio


def test_reference_run_iteration_drives_gpu_modules(ref_scheduler, lexicon):
    from paper_2211_13939_b200.modules import build_modules
    cfg = PipelineConfig()
    mods = build_modules(lexicon, cfg, tier="r", device="cuda:0")
    texts, admit_at = _script(lexicon)
    rs = ref_scheduler
    ref_reports, ref_audio = _drive(rs.RequestPool, rs.run_iteration, rs.CostModel.zero(), mods, cfg, texts, admit_at)
    our_reports, our_audio = _drive(RequestPool, run_iteration, CostModel.zero(), mods, cfg, texts, admit_at)
    assert ref_reports == our_reports
    assert not any(r[5] for r in ref_reports)
    for a, b in zip(ref_audio, our_audio):
        assert [o for o, _ in a] == [o for o, _ in b]
        for (_, x), (_, y) in zip(a, b):
            assert np.array_equal(x, y)


def test_reference_scheduler_loop_serves_gpu_modules(ref_scheduler, lexicon):
    """The reference's threaded SchedulerLoop (its own loop thread, ChunkStreams, shutdown)."""
    from paper_2211_13939_b200.modules import build_modules
    cfg = PipelineConfig()
    mods = build_modules(lexicon, cfg, tier="r", device="cuda:0")
    texts, _ = _script(lexicon)
    rs = ref_scheduler
    with rs.SchedulerLoop(mods, rs.CostModel.zero(), cfg) as loop:
        streams = [loop.submit(t)[1] for t in texts]
        chunks = [list(s) for s in streams]
    for text, cs in zip(texts, chunks):
        assert cs and cs[0].sample_offset == 0
        assert all(np.isfinite(c.samples).all() for c in cs)
