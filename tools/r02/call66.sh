#!/bin/bash
mkdir -p gpurun_out/c66
export PYTHONUNBUFFERED=1
timeout 300 python tools/loop_profile.py --qps 100 --seconds 12 --top 60 > gpurun_out/c66/lp100.txt 2>&1
