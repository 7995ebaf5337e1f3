#!/bin/bash
mkdir -p gpurun_out/c30
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py tests/test_gpu_parity_r.py -q -rf -x > gpurun_out/c30/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c30/pytest.txt
timeout 300 python tools/dec_trace.py --batches 1,24,128,256,512 --precision parity > gpurun_out/c30/trace_parity.txt 2>&1
