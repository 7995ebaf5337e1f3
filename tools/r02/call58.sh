#!/bin/bash
mkdir -p gpurun_out/c58
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py -q -rf -x -k "encoder or bilstm" > gpurun_out/c58/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c58/pytest.txt
