"""cProfile of the module calls of one serving iteration at a fixed pooled batch (host cost only).

    python tools/module_host_prof.py [--batch 24] [--reps 50]

The GPU is kept ahead with a spin before each call so host times are issue costs.
"""
import argparse
import cProfile
import pstats
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.audio import VocoderState  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=24)
ap.add_argument("--reps", type=int, default=50)
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
eng.prepare_graphs(max(64, args.batch))
lex = default_lexicon()
rng = random.Random(0)
fos = [run_frontend(random_text(rng, 150, 200, lex), lex) for _ in range(args.batch)]
encs = eng.encoder_batch(fos)
pairs = [(st, enc) for enc, st in encs]
res = eng.decoder_batch(pairs)
vst = [VocoderState.initial() for _ in pairs]
outs = eng.vocoder_batch([(v, r.mel, r.stop) for v, r in zip(vst, res)])
prof = cProfile.Profile()
for rep in range(args.reps):
    torch.cuda.synchronize()
    with torch.cuda.stream(eng.stream):
        torch.cuda._sleep(10_000_000)
    prof.enable()
    res = eng.decoder_batch(pairs)   # same states each time: cost only
    outs = eng.vocoder_batch([(v, r.mel, r.stop) for (_, v), r in zip(outs, res)])
    prof.disable()
st = pstats.Stats(prof)
st.sort_stats("tottime").print_stats(25)
