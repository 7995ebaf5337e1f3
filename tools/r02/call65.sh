#!/bin/bash
mkdir -p gpurun_out/c65
export PYTHONUNBUFFERED=1
timeout 300 python tools/iter_breakdown.py --qps 100 --seconds 12 > gpurun_out/c65/ib100.txt 2>&1
timeout 300 python tools/iter_breakdown.py --qps 100 --seconds 12 --no-consumers > gpurun_out/c65/ib100_nc.txt 2>&1
timeout 300 python tools/loop_profile.py > gpurun_out/c65/lp.txt 2>&1
