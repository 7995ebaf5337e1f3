#!/bin/bash
mkdir -p gpurun_out/c56
export PYTHONUNBUFFERED=1
for v in 0 1; do
ITTS_NO_BILSTM_TC=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_bilstm python tools/enc_time.py --batches 1,8,16,32,64,128 --lo 20 --chars 200 > gpurun_out/c56/l_$v.csv 2>&1
ITTS_NO_BILSTM_TC=$v timeout 300 python tools/enc_time.py --batches 1,8,16,32,64,128 --lo 20 --chars 200 > gpurun_out/c56/t_$v.txt 2>&1
done
