#!/bin/bash
mkdir -p gpurun_out/c62
export PYTHONUNBUFFERED=1
timeout 1800 python bench.py --side-configs 0 --no-cpu-baseline --sweep 300,350,400,450 > gpurun_out/c62/bench.txt 2>gpurun_out/c62/bench.err; echo "rc $?" >> gpurun_out/c62/bench.err
