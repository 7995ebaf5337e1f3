#!/bin/bash
mkdir -p gpurun_out/c47
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/c47/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c47/pytest.txt
timeout 300 python tools/iter_breakdown.py --qps 300 --seconds 10 > gpurun_out/c47/iter_300.txt 2>&1
timeout 300 python tools/soak.py --qps 250 --seconds 60 > gpurun_out/c47/soak_250.txt 2>&1; echo "rc $?" >> gpurun_out/c47/soak_250.txt
