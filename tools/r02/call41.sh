#!/bin/bash
mkdir -p gpurun_out/c41
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py -q -rf -x -k "encoder" > gpurun_out/c41/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c41/pytest.txt
timeout 300 python tools/enc_time.py --batches 1,8,16,64,128 --chars 200 > gpurun_out/c41/enc_time.txt 2>&1
timeout 300 python tools/enc_time.py --batches 1,16,128 --chars 110 >> gpurun_out/c41/enc_time.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_bilstm python tools/enc_time.py --batches 8,16,128 --chars 200 > gpurun_out/c41/launches.csv 2>&1
