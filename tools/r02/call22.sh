#!/bin/bash
mkdir -p gpurun_out/c22
for p in parity bf16; do
timeout 300 python tools/dec_trace.py --batches 1,24,64,128,256 --precision $p > gpurun_out/c22/trace_$p.txt 2>&1
done
