"""cProfile of the host side of one serving iteration at a fixed pooled batch: an encoder call for
`--new` fresh requests, then a decoder and a vocoder call for `--batch` items.  The GPU is kept
busy with a long sleep before each call, so the times are issue / host costs only.

    python tools/module_host_prof.py [--batch 285] [--new 8] [--reps 20]
"""
import argparse
import cProfile
import pstats
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.audio import VocoderState  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=285)
ap.add_argument("--new", type=int, default=8)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
eng.prepare_graphs(min(512, max(64, args.batch)))
lex = default_lexicon()
rng = random.Random(0)
fos = [run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(args.batch)]
new_fos = [run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(args.new)]
encs = eng.encoder_batch(fos)
pairs = [(st, enc) for enc, st in encs]
res = eng.decoder_batch(pairs)
vst = [VocoderState.initial() for _ in pairs]
outs = eng.vocoder_batch([(v, r.mel, False) for v, r in zip(vst, res)])
eng.encoder_batch(new_fos)
torch.cuda.synchronize()
prof = cProfile.Profile()
wall = {"E": 0.0, "D": 0.0, "V": 0.0}
for rep in range(args.reps):
    torch.cuda.synchronize()
    with torch.cuda.stream(eng.stream):
        torch.cuda._sleep(50_000_000)
    prof.enable()
    t = time.perf_counter()
    eng.encoder_batch(new_fos)
    t1 = time.perf_counter()
    res = eng.decoder_batch(pairs)   # same states each time: cost only
    t2 = time.perf_counter()
    prof.disable()
    wall["E"] += t1 - t
    wall["D"] += t2 - t1
    torch.cuda.synchronize()
    with torch.cuda.stream(eng.stream):
        torch.cuda._sleep(50_000_000)
    prof.enable()
    t = time.perf_counter()
    eng.idle_hook = lambda done, t0=time.perf_counter(): None
    outs = eng.vocoder_batch([(v, r.mel, False) for (_, v), r in zip(outs, res)])
    prof.disable()
    wall["V"] += time.perf_counter() - t
print({k: round(1e3 * v / args.reps, 3) for k, v in wall.items()}, "ms per call (V includes the GPU wait)")
st = pstats.Stats(prof)
st.sort_stats("tottime").print_stats(30)
