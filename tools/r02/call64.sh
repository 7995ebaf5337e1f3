#!/bin/bash
mkdir -p gpurun_out/c64
export PYTHONUNBUFFERED=1
timeout 600 python tools/module_times.py --batches 8,12,14,15,16,17,18,20,24,28,32,48,64 --reps 20 > gpurun_out/c64/mt.txt 2>&1
