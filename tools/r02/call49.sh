#!/bin/bash
mkdir -p gpurun_out/c49
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/test_gpu_tier_r.py tests/test_gpu_parity_r.py tests/test_gpu_reference_dropin.py -q -rf -x > gpurun_out/c49/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c49/pytest.txt
timeout 300 python tools/iter_breakdown.py --qps 300 --seconds 10 > gpurun_out/c49/iter_300.txt 2>&1
timeout 1500 python bench.py --sweep 275,325,375 --side-configs 0 --no-cpu-baseline > gpurun_out/c49/bench.txt 2>gpurun_out/c49/bench.err; echo "rc $?" >> gpurun_out/c49/bench.err
