#!/bin/bash
mkdir -p gpurun_out/c28
export PYTHONUNBUFFERED=1
timeout 600 python tools/module_host_prof.py --batch 512 --reps 5 > gpurun_out/c28/hostprof512.txt 2>&1
timeout 600 python tools/module_host_prof.py --batch 128 --reps 10 > gpurun_out/c28/hostprof128.txt 2>&1
