#!/bin/bash
mkdir -p gpurun_out/c26
export PYTHONUNBUFFERED=1
timeout 1200 python bench.py > gpurun_out/c26/bench.txt 2>gpurun_out/c26/bench.err; echo "rc $?" >> gpurun_out/c26/bench.err
