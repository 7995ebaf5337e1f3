#!/bin/bash
mkdir -p gpurun_out/c54
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py -q -rf -x -k "encoder or end_to_end" > gpurun_out/c54/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c54/pytest.txt
timeout 300 python tools/enc_time.py --batches 1,8,16,64,128 --lo 20 --chars 200 > gpurun_out/c54/enc_time.txt 2>&1
