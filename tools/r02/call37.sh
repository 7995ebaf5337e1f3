#!/bin/bash
mkdir -p gpurun_out/c37
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/c37/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c37/pytest.txt
for i in 1 2; do
  timeout 300 python tools/soak.py --qps 200 --seconds 60 > gpurun_out/c37/soak_$i.txt 2>&1; echo "rc $?" >> gpurun_out/c37/soak_$i.txt
done
for q in 100 270; do
timeout 300 python tools/iter_breakdown.py --qps $q --seconds 10 > gpurun_out/c37/iter_$q.txt 2>&1
done
