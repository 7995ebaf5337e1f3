"""Per-phase time breakdown of the persistent decoder kernel (itts_r_decode_debug_trace).

    python tools/dec_trace.py [--batches 16,64,128]
"""
import argparse
import random
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200 import _native  # noqa: E402
from paper_2211_13939_b200.domain import PipelineConfig  # noqa: E402
from paper_2211_13939_b200.frontend import default_lexicon, run_frontend  # noqa: E402
from paper_2211_13939_b200.harness import random_text  # noqa: E402
from paper_2211_13939_b200.tier_r import TierREngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="16,64,128")
ap.add_argument("--precision", default="parity")
args = ap.parse_args()
eng = TierREngine(PipelineConfig(), "cuda:0")
eng.use_graphs = False
eng.set_precision(args.precision)
lex = default_lexicon()
names = ["PRE", "ATT gates+q", "ATT-A", "ATT-B (or DEC gates+combine+proj)", "DEC gates+proj"]
for B in [int(x) for x in args.batches.split(",")]:
    rng = random.Random(B)
    fos = [run_frontend(random_text(rng, 20, 200, lex), lex) for _ in range(B)]
    encs = eng.encoder_batch(fos)
    eng.decoder_batch([(st, enc) for enc, st in encs])
    torch.cuda.synchronize()
    buf = torch.zeros(32, dtype=torch.int64, device="cuda")
    _native.call("itts_r_decode_debug_trace", buf.data_ptr())
    REPS = 4
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    for _ in range(REPS):
        eng.decoder_batch([(st, enc) for enc, st in encs])
    e1.record(eng.stream)
    torch.cuda.synchronize()
    _native.call("itts_r_decode_debug_trace", None)
    raw = buf.cpu().tolist()
    t = raw[:5] + [v / REPS for v in raw[5:]]   # phase totals are per launch (last one); the rest accumulate
    # phases per step: PRE overlapped with the attention gates for B <= 40 (148 SMs), no barrier
    # between ATT-A and the decoder gates for B <= 96 (merged combine, per-item chunk counters)
    prem, merged = B <= 40, B <= 96
    if merged:   # one grid barrier per step after the decoder gates (+ one after PRE if not overlapped)
        nm = (["whole step"] if prem else ["PRE", "ATT gates + ATT-A + DEC gates"])
    else:
        nm = ["PRE", "ATT gates+q", "ATT-A", "ATT-B", "DEC gates+proj"]
    nm += ["-"] * (5 - len(nm))
    print(f"B={B}: chunk {e0.elapsed_time(e1) / REPS:.3f} ms; per step (us): " +
          ", ".join(f"{n} {t[i] / 32e3:.1f}" for i, n in enumerate(nm) if t[i]))
    print(f"   PRE first PRE CTA (us): mel partials {t[5] / 32e3:.2f}, H1 {t[6] / 32e3:.2f}, p gemv {t[7] / 32e3:.2f}"
          + (f"; overlapped: start {t[15] / 31e3:.2f}, released {t[14] / 31e3:.2f} after the CTA's barrier" if t[14] else ""))
    for m, nm in ((0, "ATT"), (1, "DEC")):
        g = [t[16 + 8 * m + i] / 32e3 for i in range(7)]
        print(f"   {nm} gates CTA0 (us from phase start): producer issued {g[0]:.1f}, first stage {g[1]:.1f}, "
              f"MMA done {g[2]:.1f}, acc ready {g[3]:.1f}, group synced {g[4]:.1f}, cells {g[6]:.1f}, partials {g[5]:.1f}")
    if t[13]:
        sub = ["next-task issue", "bulk wait", "energies", "softmax+next MMA", "context"]
        print(f"   ATT-A CTA0: {t[13] / 32:.1f} tasks/step; per task (us): " +
              ", ".join(f"{n} {t[8 + i] / t[13] / 1e3:.2f}" for i, n in enumerate(sub)))
