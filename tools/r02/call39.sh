#!/bin/bash
mkdir -p gpurun_out/c39
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py tests/test_gpu_parity_r.py -q -rf -x > gpurun_out/c39/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c39/pytest.txt
timeout 300 python tools/enc_time.py --batches 1,8,16,64,128 --chars 200 > gpurun_out/c39/enc_time.txt 2>&1
timeout 300 python tools/enc_time.py --batches 1,16,128 --chars 110 >> gpurun_out/c39/enc_time.txt 2>&1
