#!/bin/bash
mkdir -p gpurun_out/c42
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py -q -rf -x -k "encoder" > gpurun_out/c42/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c42/pytest.txt
for g in 1 2 4 8 16; do
echo "G=$g" >> gpurun_out/c42/enc_time.txt
ITTS_BILSTM_G=$g timeout 300 python tools/enc_time.py --batches 16,64,128 --lo 20 --chars 200 >> gpurun_out/c42/enc_time.txt 2>&1
done
