#!/bin/bash
mkdir -p gpurun_out/c55
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bilstm_tc -c 1 -o gpurun_out/c55/bt128 python tools/enc_time.py --batches 128 --lo 20 --chars 200 > gpurun_out/c55/ncu.log 2>&1
