#!/bin/bash
mkdir -p gpurun_out/c27
export PYTHONUNBUFFERED=1
timeout 600 python tools/module_times.py --batches 24,128,256,512 > gpurun_out/c27/module_times.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c27/launches_b512.csv python tools/profile_iter.py --batches 512 --iters 2 > /dev/null 2>&1
