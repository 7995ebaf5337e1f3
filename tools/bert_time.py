"""Device time of the BERT prosody frontend (f4) for pooled batches of texts.

    python tools/bert_time.py [--batches 1,3,8,32] [--chars 110]
"""
import argparse
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200.bert_frontend import FFN, HIDDEN, LAYERS, BertProsody  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,3,8,32")
ap.add_argument("--chars", type=int, default=110)
args = ap.parse_args()
lex = default_lexicon()
bert = BertProsody(lex, "cuda:0")
macs_per_char = LAYERS * (4 * HIDDEN * HIDDEN + 2 * HIDDEN * FFN)
for B in [int(x) for x in args.batches.split(",")]:
    rng = random.Random(B)
    texts = [random_text(rng, args.chars, args.chars, lex) for _ in range(B)]
    bert.run(texts)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(bert.stream)
        bert.run(texts)
        e1.record(bert.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    rows = sum(len(t) for t in texts)
    ms = min(ts)
    print(f"B={B} chars={rows}: {ms:.3f} ms (incl. H2D/D2H), {2 * macs_per_char * rows / ms / 1e9:.1f} TFLOP/s GEMM",
          flush=True)
