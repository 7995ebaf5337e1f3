#!/bin/bash
mkdir -p gpurun_out/c46
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py -q -rf -x > gpurun_out/c46/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c46/pytest.txt
