"""Host-time breakdown of one decoder_batch call (graph path): entry, items, plan, replay, results."""
import sys, random, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2211_13939_b200.tier_r as tr
from paper_2211_13939_b200.audio import VocoderState
from paper_2211_13939_b200.domain import PipelineConfig
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend
from paper_2211_13939_b200.harness import random_text
eng = tr.TierREngine(PipelineConfig(), "cuda:0")
eng.prepare_graphs(64)
lex = default_lexicon()
rng = random.Random(0)
fos = [run_frontend(random_text(rng, 150, 200, lex), lex) for _ in range(16)]
live = [(enc, st, VocoderState.initial()) for enc, st in eng.encoder_batch(fos)]
# instrument: wrap graph.replay and _dec_items
marks = []
orig_items = eng._dec_items
def items(*a, **k):
    marks.append(("items0", time.perf_counter())); r = orig_items(*a, **k); marks.append(("items1", time.perf_counter())); return r
eng._dec_items = items
import torch.cuda.graphs as G
orig_replay = G.CUDAGraph.replay
def replay(self):
    marks.append(("replay0", time.perf_counter())); orig_replay(self); marks.append(("replay1", time.perf_counter()))
G.CUDAGraph.replay = replay
res_t = []
for it in range(40):
    marks.clear()
    t0 = time.perf_counter()
    res = eng.decoder_batch([(st, enc) for enc, st, _ in live])
    t1 = time.perf_counter()
    marks.append(("end", t1))
    outs = eng.vocoder_batch([(vs, r.mel, r.stop) for (_, _, vs), r in zip(live, res)])
    live = [(enc, r.state, vs) for (enc, _, _), r, (_, vs) in zip(live, res, outs) if not r.stop]
    d = {}
    for k, v in marks:
        d.setdefault(k, v)   # first occurrence: inside decoder_batch (the vocoder's speculation comes later)
    if it > 5 and "replay0" in d and d["items0"] < d["end"]:
        res_t.append((1e6*(d["items0"]-t0), 1e6*(d["items1"]-d["items0"]), 1e6*(d["replay0"]-d["items1"]), 1e6*(d["replay1"]-d["replay0"]), 1e6*(t1-d["replay1"])))
    if not live: break
a = np.array(res_t)
print("median us: entry->items %.1f, items %.1f, items->replay %.1f, replay %.1f, after %.1f" % tuple(np.median(a, 0)))
