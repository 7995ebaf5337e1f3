#!/bin/bash
# x2 parity products (bf16-grid weights), B <= 512 persistent decoder, shared bucket scratch
mkdir -p gpurun_out/c23
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_decoder_paths.py tests/test_gpu_parity_r.py -q -rf -x > gpurun_out/c23/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c23/pytest.txt
for p in parity bf16; do
timeout 300 python tools/dec_trace.py --batches 1,24,128,256,384,512 --precision $p > gpurun_out/c23/trace_$p.txt 2>&1
done
