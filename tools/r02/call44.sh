#!/bin/bash
mkdir -p gpurun_out/c44
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py tests/test_gpu_parity_r.py -q -rf -x > gpurun_out/c44/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c44/pytest.txt
timeout 300 python tools/enc_time.py --batches 1,8,16 --lo 20 --chars 200 > gpurun_out/c44/enc_time.txt 2>&1
timeout 1500 python bench.py > gpurun_out/c44/bench.txt 2>gpurun_out/c44/bench.err; echo "rc $?" >> gpurun_out/c44/bench.err
