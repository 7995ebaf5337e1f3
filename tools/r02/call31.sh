#!/bin/bash
mkdir -p gpurun_out/c31
export PYTHONUNBUFFERED=1
timeout 600 python tools/loop_profile.py --qps 240 --seconds 12 > gpurun_out/c31/loopprof240.txt 2>&1
