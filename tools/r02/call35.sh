#!/bin/bash
mkdir -p gpurun_out/c35
export PYTHONUNBUFFERED=1
timeout 600 python tools/module_host_prof.py --batch 285 --new 8 --reps 20 > gpurun_out/c35/hostprof.txt 2>&1
