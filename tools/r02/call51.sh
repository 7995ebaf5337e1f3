#!/bin/bash
mkdir -p gpurun_out/c51
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tc_conv.py tests/test_gpu_tier_r.py tests/test_gpu_resblock.py -q -rf -x > gpurun_out/c51/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c51/pytest.txt
timeout 300 python tools/module_times.py --batches 16,230 > gpurun_out/c51/times.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_conv_tc python tools/profile_iter.py --batches 230 --iters 1 > gpurun_out/c51/convs.csv 2>&1
