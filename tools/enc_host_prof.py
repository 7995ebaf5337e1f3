"""cProfile of encoder_batch (+ the frontend) host cost for a few new requests per call.

    python tools/enc_host_prof.py [--items 2] [--reps 50]
"""
import argparse
import cProfile
import pstats
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
ap.add_argument("--items", type=int, default=2)
ap.add_argument("--reps", type=int, default=50)
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
lex = default_lexicon()
rng = random.Random(0)
texts = [[random_text(rng, 20, 200, lex) for _ in range(args.items)] for _ in range(args.reps)]
eng.encoder_batch([run_frontend(t, lex) for t in texts[0]])
torch.cuda.synchronize()
prof = cProfile.Profile()
keep = []
for rep in range(args.reps):
    with torch.cuda.stream(eng.stream):
        torch.cuda._sleep(5_000_000)
    prof.enable()
    fos = [run_frontend(t, lex) for t in texts[rep]]
    keep.append(eng.encoder_batch(fos))
    prof.disable()
    torch.cuda.synchronize()
pstats.Stats(prof).sort_stats("cumulative").print_stats(30)
