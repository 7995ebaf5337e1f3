"""Is the vocoder call host-bound at small pooled batches?

    python tools/voc_hostbound.py [--batches 1,8,24,64]

Times vocoder_batch on the engine stream twice per batch: as served (host
issues the launches while the GPU runs them) and queued behind a 20 ms GPU
spin, so every launch is issued before the first one starts (pure device
time).  The difference is host issue time the GPU waits for.  Both MRF modes
(three streams / serial).
"""

import argparse
import json
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2211_13939_b200.audio import VocoderState  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,8,24,64")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    eng = TierREngine(PipelineConfig(), "cuda:0")
    lex = default_lexicon()
    for B in [int(b) for b in args.batches.split(",")]:
        rng = random.Random(B)
        fos = [run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(B)]
        encs = eng.encoder_batch(fos)
        res = eng.decoder_batch([(st, enc) for enc, st in encs])
        triples = [(VocoderState.initial(), r.mel, False) for r in res]
        row = {"B": B}
        for streams in (True, False):
            eng.mrf_streams = streams
            for queued in (False, True):
                ts, hs = [], []
                for _ in range(args.reps + 1):
                    torch.cuda.synchronize()
                    if queued:
                        with torch.cuda.stream(eng.stream):
                            torch.cuda._sleep(40_000_000)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(eng.stream)
                    t0 = time.perf_counter()
                    eng.vocoder_batch(triples)
                    hs.append((time.perf_counter() - t0) * 1e3)
                    e1.record(eng.stream)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                key = ("streams" if streams else "serial") + ("_queued" if queued else "")
                row[key] = round(sorted(ts[1:])[len(ts) // 2 - 1], 3)
                if queued:
                    row[key + "_host_ms"] = round(sorted(hs[1:])[len(hs) // 2 - 1] - 0, 3)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
