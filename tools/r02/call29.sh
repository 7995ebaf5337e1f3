#!/bin/bash
mkdir -p gpurun_out/c29
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py -q -rf -x > gpurun_out/c29/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c29/pytest.txt
timeout 300 python tools/dec_trace.py --batches 1,24,128,256,512 --precision parity > gpurun_out/c29/trace_parity.txt 2>&1
