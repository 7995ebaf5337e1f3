#!/bin/bash
mkdir -p gpurun_out/c43
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py tests/test_gpu_resblock.py -q -rf -x > gpurun_out/c43/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c43/pytest.txt
for q in 100 300; do
timeout 300 python tools/iter_breakdown.py --qps $q --seconds 10 > gpurun_out/c43/iter_$q.txt 2>&1
done
