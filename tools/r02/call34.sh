#!/bin/bash
mkdir -p gpurun_out/c34
export PYTHONUNBUFFERED=1
for q in 100 240 270; do
timeout 300 python tools/iter_breakdown.py --qps $q --seconds 10 > gpurun_out/c34/iter_$q.txt 2>&1
done
