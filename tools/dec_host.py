"""Host-side cost of one decoder_batch call (graph replay vs eager persistent launch).

    python tools/dec_host.py [--batches 1,24,64]

The GPU is kept busy with a long spin first, so the measured host time is pure
issue cost (plan building, H2D, launches), not waiting.
"""
import argparse
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,24,64")
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
lex = default_lexicon()
for B in [int(x) for x in args.batches.split(",")]:
    rng = random.Random(B)
    fos = [run_frontend(random_text(rng, 60, 200, lex), lex) for _ in range(B)]
    pairs = [(st, enc) for enc, st in eng.encoder_batch(fos)]
    row = {}
    for graphs in (True, False):
        eng.use_graphs = graphs
        eng.decoder_batch(pairs)
        hs, ds = [], []
        for _ in range(6):
            torch.cuda.synchronize()
            with torch.cuda.stream(eng.stream):
                torch.cuda._sleep(20_000_000)
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
            eng.decoder_batch(pairs)
            e1.record(eng.stream)
            hs.append((time.perf_counter() - t0) * 1e3)
            torch.cuda.synchronize()
            ds.append(e0.elapsed_time(e1))
        row["graph" if graphs else "eager"] = dict(host_ms=round(sorted(hs)[3], 3), dev_ms=round(sorted(ds)[3], 3))
    print(B, row, flush=True)
