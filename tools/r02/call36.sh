#!/bin/bash
mkdir -p gpurun_out/c36
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py -q -rf -x > gpurun_out/c36/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c36/pytest.txt
for q in 100 270; do
timeout 300 python tools/iter_breakdown.py --qps $q --seconds 10 > gpurun_out/c36/iter_$q.txt 2>&1
done
