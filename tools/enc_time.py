"""Device time of encoder_batch (embedding, convs, BiLSTM, processed memory) for a few new items.

    python tools/enc_time.py [--batches 1,3,8] [--chars 200]
"""
import argparse
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,3,8")
ap.add_argument("--chars", type=int, default=200)
ap.add_argument("--lo", type=int, default=None, help="ragged texts: U{lo..chars} characters")
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
lex = default_lexicon()
for B in [int(x) for x in args.batches.split(",")]:
    rng = random.Random(B)
    fos = [run_frontend(random_text(rng, args.lo or args.chars, args.chars, lex), lex) for _ in range(B)]
    eng.encoder_batch(fos)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        eng.encoder_batch(fos)
        e1.record(eng.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    L = max(len(f.phonemes) for f in fos)
    print(f"B={B} L_max={L}: encoder {min(ts):.3f} ms", flush=True)
