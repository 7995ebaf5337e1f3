#!/bin/bash
mkdir -p gpurun_out/c32
export PYTHONUNBUFFERED=1
timeout 1200 python bench.py --sweep 240,275,300,325 --side-configs 0 --no-cpu-baseline > gpurun_out/c32/bench.txt 2>gpurun_out/c32/bench.err; echo "rc $?" >> gpurun_out/c32/bench.err
