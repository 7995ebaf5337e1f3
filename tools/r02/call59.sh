#!/bin/bash
mkdir -p gpurun_out/c59
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/c59/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c59/pytest.txt
timeout 300 python tools/iter_breakdown.py --qps 100 --seconds 10 > gpurun_out/c59/iter_100.txt 2>&1
timeout 1500 python bench.py --side-configs 0 --no-cpu-baseline --sweep 275,330,375 > gpurun_out/c59/bench.txt 2>gpurun_out/c59/bench.err; echo "rc $?" >> gpurun_out/c59/bench.err
