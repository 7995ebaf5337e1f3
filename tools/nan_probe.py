"""Debug aid: serve under Poisson load and report the first module call that produced non-finite
values (decoder mel checked right before the vocoder runs, vocoder audio by the module itself).

    python tools/nan_probe.py [--qps 150] [--runs 3]
"""
import argparse
import collections
import gc
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon  # noqa: E402
from paper_2211_13939_b200.harness import TimedRequest, poisson_trace, random_text, serve  # noqa: E402
from paper_2211_13939_b200.modules import build_engine, modules_for  # noqa: E402
from paper_2211_13939_b200.scheduler import PipelineModules  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--qps", type=float, default=150)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--sync", action="store_true")
ap.add_argument("--seed", type=int, default=150)
args = ap.parse_args()
cfg, lex = PipelineConfig(), default_lexicon()
eng = build_engine(cfg, "r", "cuda:0")
eng.prepare_graphs(max_batch=256)
base = modules_for(eng, lex)
state = {"first": None, "calls": 0}


SYNC = "--sync" in sys.argv


def voc(triples):
    state["calls"] += 1
    if state["first"] is None and SYNC:
        torch.cuda.synchronize()
        bad = [i for i, (_, m, _) in enumerate(triples) if not torch.isfinite(m.data).all()]
        if bad:
            state["first"] = (f"call {state['calls']}: mel non-finite for {len(bad)}/{len(triples)} items "
                              f"(first {bad[:4]}, frames {[triples[i][1].frame_count for i in bad[:4]]}, "
                              f"L {[triples[i][1].req.seq_len for i in bad[:4]]})")
    try:
        return base.vocoder_batch(triples)
    except Exception as exc:  # noqa: BLE001
        if state["first"] is None:
            bad = [i for i, (_, m, _) in enumerate(triples) if not torch.isfinite(m.data).all()]
            tails = [i for i, (vs, _, _) in enumerate(triples)
                     if getattr(vs, "has_tail", False) and not torch.isfinite(
                         eng.arena.tensor[vs.buf.off:vs.buf.off + eng.voc_size()]).all()]
            state["first"] = (f"call {state['calls']}: vocoder raised {exc}; B={len(triples)}; mel non-finite "
                              f"items {bad[:6]} of {len(bad)}; tail non-finite {tails[:6]} of {len(tails)}; "
                              f"frames {[t[1].frame_count for t in triples][:8]}")
        raise


mods = PipelineModules(base.frontend_batch, base.encoder_batch, base.decoder_batch, voc)
wr = random.Random(8)
for burst in (8, 32, 64):
    serve(mods, cfg, [TimedRequest(0.0, random_text(wr, 20, 200, lex)) for _ in range(burst)], warmup_iters=0,
          timed_iters=None, drain_seconds=0.0)
gc.collect()
gc.freeze()
gc.set_threshold(200000, 100, 100)
for r in range(args.runs):
    run = serve(mods, cfg, poisson_trace(args.qps, 12, seed=args.seed + r, lexicon=lex), warmup_iters=3, warmup_seconds=1.0,
                timed_iters=None, timed_seconds=10, drain_seconds=2.0, tail_seconds=10)
    errs = collections.Counter(r.error for r in run.timings if r.error)
    print(f"run {r}: failed {sum(errs.values())}; first: {state['first']}", flush=True)
