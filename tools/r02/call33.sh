#!/bin/bash
mkdir -p gpurun_out/c33
export PYTHONUNBUFFERED=1
timeout 600 python tools/loop_profile.py --qps 270 --seconds 12 > gpurun_out/c33/loopprof270.txt 2>&1
