import sys, random, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2211_13939_b200.tier_r as tr
from paper_2211_13939_b200.domain import PipelineConfig
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend
from paper_2211_13939_b200.harness import random_text
eng = tr.TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = False
lex = default_lexicon()
for B in (160, 192, 224, 256):
    rng = random.Random(B)
    fos = [run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(B)]
    pairs = [(st, enc) for enc, st in eng.encoder_batch(fos)]
    row = {}
    for limit in (192, 256):
        tr.PERSIST_MAX_B = limit
        eng.decoder_batch(pairs)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream); eng.decoder_batch(pairs); e1.record(eng.stream); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row[limit] = round(min(ts), 3)
    print(B, row, flush=True)
