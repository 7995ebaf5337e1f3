#!/bin/bash
mkdir -p gpurun_out/c38
export PYTHONUNBUFFERED=1
timeout 1500 python bench.py --sweep 275,325,375,425 --side-configs 0 --no-cpu-baseline > gpurun_out/c38/bench.txt 2>gpurun_out/c38/bench.err; echo "rc $?" >> gpurun_out/c38/bench.err
