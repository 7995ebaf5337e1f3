#!/bin/bash
mkdir -p gpurun_out/c40
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bilstm_g -c 1 -o gpurun_out/c40/prof_bilstm_g python tools/enc_time.py --batches 128 --chars 200 > gpurun_out/c40/ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__cluster_max_active_clusters,launch__grid_size --clock-control none --csv -k regex:k_bilstm python tools/enc_time.py --batches 8,16,128 --chars 200 > gpurun_out/c40/launches.csv 2>&1
