"""Per-module device/host time of one serving iteration at several pooled batch sizes.

    python tools/profile_iter.py [--tier r] [--batches 1,16,64,128,256]

Builds B requests of U{20..200} chars (seeded), runs them through the
module calls exactly like run_iteration (F, E on new items, then D, V on
all), and reports per-call wall time (host, includes sync for V) and the
device time between CUDA events on the engine stream.
"""

from __future__ import annotations

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
from paper_2211_13939_b200.modules import build_engine  # noqa: E402


def texts(n, seed, lo=20, hi=200):
    lex = default_lexicon()
    singles = sorted(c for c in lex.phrase_to_pinyin if len(c) == 1)
    rng = random.Random(seed)
    return ["".join(rng.choice(singles) for _ in range(rng.randint(lo, hi))) for _ in range(n)]


def timed(engine, fn, *args):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0.record(engine.stream)
    out = fn(*args)
    ev1.record(engine.stream)
    t1 = time.perf_counter()
    ev1.synchronize()
    return out, (t1 - t0) * 1e3, ev0.elapsed_time(ev1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tier", default="r")
    ap.add_argument("--batches", default="1,16,64,128,256")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--no-graphs", action="store_true", help="eager decoder (stable kernel order for ncu -s/-c)")
    ap.add_argument("--unfused", action="store_true", help="MRF as two tc_conv launches per layer (A/B)")
    ap.add_argument("--serial-mrf", action="store_true", help="MRF branches one after another on one stream")
    ap.add_argument("--postnet", action="store_true", help="chunk-local PostNet on the decoder output (f3)")
    args = ap.parse_args()
    cfg = PipelineConfig()
    eng = build_engine(cfg, args.tier, "cuda:0")
    if args.no_graphs:
        eng.use_graphs = False
    if args.unfused:
        eng.fused_mrf = False
    if args.serial_mrf:
        eng.mrf_streams = False
    if args.postnet:
        eng.set_postnet(True)
    lex = default_lexicon()
    rows = []
    for B in [int(b) for b in args.batches.split(",")]:
        fos = [run_frontend(t, lex) for t in texts(B, B)]
        (encs, e_host, e_dev) = timed(eng, eng.encoder_batch, fos)
        live = [(enc, st, VocoderState.initial()) for enc, st in encs]
        for it in range(args.iters):
            l0 = eng.launches
            res, d_host, d_dev = timed(eng, eng.decoder_batch, [(st, enc) for enc, st, _ in live])
            outs, v_host, v_dev = timed(eng, eng.vocoder_batch,
                                        [(vs, r.mel, r.stop) for (_, _, vs), r in zip(live, res)])
            launches = eng.launches - l0
            live = [(enc, r.state, vs) for (enc, _, _), r, (_, vs) in zip(live, res, outs) if not r.stop]
        frames = sum(r.mel.frame_count + (4 if it else 0) for r in res)
        rows.append(dict(B=B, enc_host_ms=round(e_host, 2), enc_dev_ms=round(e_dev, 2),
                         dec_host_ms=round(d_host, 2), dec_dev_ms=round(d_dev, 2),
                         voc_host_ms=round(v_host, 2), voc_dev_ms=round(v_dev, 2),
                         launches=launches, voc_frames=frames,
                         voc_tflops=round(2 * 307.05e6 * frames / (v_dev * 1e-3) / 1e12, 1)))
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
