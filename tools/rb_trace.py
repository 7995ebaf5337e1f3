"""Barrier-wait breakdown of the fused ResBlock kernel (itts_resblock_debug_trace).

    python tools/rb_trace.py [--rows 295000] [--c 128] [--k 3] [--dil 1]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2211_13939_b200 import _native, tc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=295000)
ap.add_argument("--c", type=int, default=128)
ap.add_argument("--k", type=int, default=3)
ap.add_argument("--dil", type=int, default=1)
args = ap.parse_args()
C, k = args.c, args.k
dev = "cuda:0"
x = (torch.randn(args.rows, C, device=dev) * 0.5).to(torch.bfloat16)
w = (torch.randn(k, C, C, device=dev) / (C * k) ** 0.5).to(torch.bfloat16)
b = torch.zeros(C, device=dev)
ro = torch.arange(args.rows, dtype=torch.int32, device=dev)
out = torch.empty_like(x)
layer = (w, [0] * k, b)
for _ in range(3):
    tc.resblock_tc(x, layer, layer, args.dil, ro, act_out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    tc.resblock_tc(x, layer, layer, args.dil, ro, act_out=out)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 100
macs = 2 * args.rows * C * C * k
print(f"C={C} k={k} dil={args.dil} rows={args.rows}: {us:.1f} us/launch, {2 * macs / us / 1e6:.1f} TFLOP/s")
buf = torch.zeros(2 * 148, 16, dtype=torch.int64, device=dev)  # up to 2 CTAs per SM
_native.call("itts_resblock_debug_trace", buf.data_ptr())
tc.resblock_tc(x, layer, layer, args.dil, ro, act_out=out)
torch.cuda.synchronize()
_native.call("itts_resblock_debug_trace", None)
t = buf[buf[:, 7] > 0].double().mean(0).cpu()
tot = t[7].item()
names = ["mma: x_full", "mma: a1_empty", "mma: w_full c1", "mma: a2_empty", "mma: t_ready", "mma: w_full c2", "-",
         "mma: total", "epi: a1_full", "epi: t_empty", "epi: epi1 work", "epi: a2_full", "epi: r_full",
         "epi: epi2 work", "epi: bar", "-"]
for n, v in zip(names, t.tolist()):
    if n != "-":
        print(f"  {n:18s} {v:12.0f} cyc  {100 * v / tot:5.1f}%")
