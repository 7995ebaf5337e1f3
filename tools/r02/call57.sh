#!/bin/bash
mkdir -p gpurun_out/c57
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py -q -rf -x -k "encoder or end_to_end" > gpurun_out/c57/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c57/pytest.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_bilstm python tools/enc_time.py --batches 1,8,16,32,64,128 --lo 20 --chars 200 > gpurun_out/c57/l.csv 2>&1
