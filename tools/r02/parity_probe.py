"""Mel error growth of the GPU decoder vs the fp32 oracle over long requests (solo decoding).

    python tools/r02/parity_probe.py [--chars 50,200,1000]
"""
import argparse
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import tier_r as orc  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402
from paper_2211_13939_b200.weights import tier_r_weights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--chars", default="50,200,1000")
ap.add_argument("--precision", default=None)
ap.add_argument("--oracle-encoder", action="store_true", help="feed the oracle's fp32 memory / processed memory")
args = ap.parse_args()
torch.set_num_threads(len(__import__("os").sched_getaffinity(0)))
w = tier_r_weights(0)
eng = TierREngine(PipelineConfig(), "cuda:0", weights=w)
if args.precision:
    eng.set_precision(args.precision)
lex = default_lexicon()
rng = random.Random(0)
for n in [int(x) for x in args.chars.split(",")]:
    text = random_text(rng, n, n, lex)
    fo = run_frontend(text, lex)
    (enc, st), = eng.encoder_batch([fo])
    m_o, pm_o = orc.encode(w, fo.phonemes, fo.pw, fo.pph, fo.iph)
    print(f"  encoder max-abs: memory {np.abs(enc.rows - m_o.numpy()).max():.3e} processed "
          f"{np.abs(eng.read_processed_memory(enc.req) - pm_o.numpy()).max():.3e}", flush=True)
    if args.oracle_encoder:
        m_o, pm_o = orc.encode(w, fo.phonemes, fo.pw, fo.pph, fo.iph)
        t = eng.arena.tensor
        eng.stream.synchronize()
        t[enc.req.extra["mem_off"]:enc.req.extra["mem_off"] + m_o.numel()].copy_(m_o.reshape(-1).to(t.device))
        t[enc.req.extra["pm_off"]:enc.req.extra["pm_off"] + pm_o.numel()].copy_(pm_o.reshape(-1).to(t.device))
        torch.cuda.synchronize()
    gpu = []
    while True:
        r, = eng.decoder_batch([(st, enc)])
        gpu.append(r.mel.frames)
        st = r.state
        if r.stop:
            break
    gpu = np.concatenate(gpu)
    t0 = time.time()
    mem, pm = orc.encode(w, fo.phonemes, fo.pw, fo.pph, fo.iph)
    s = orc.init_state(mem.shape[0], 8)
    ref = []
    while True:
        m, stop, s, _ = orc.decode_chunk(w, s, mem, pm, 32)
        ref.append(m.numpy())
        if stop:
            break
    ref = np.concatenate(ref)
    err = np.abs(gpu - ref)
    per_chunk = [float(err[i:i + 32].max()) for i in range(0, len(err), 32)]
    marks = [0, 1, 3, 7, 15, 31, 63, 127, 255, 511]
    print(f"{n} chars: L={fo.seq_len} frames={len(ref)} oracle {time.time() - t0:.0f}s  max-abs {err.max():.3e}  "
          f"mean-abs {err.mean():.3e}  |ref| max {np.abs(ref).max():.3f}", flush=True)
    print("  per-chunk max err at chunks", {k: f"{per_chunk[k]:.2e}" for k in marks if k < len(per_chunk)}, flush=True)
