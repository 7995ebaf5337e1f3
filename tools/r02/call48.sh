#!/bin/bash
mkdir -p gpurun_out/c48
export PYTHONUNBUFFERED=1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c48/smoke.txt 2>&1; echo "rc $?" >> gpurun_out/c48/smoke.txt
timeout 1800 python bench.py > gpurun_out/c48/bench.txt 2>gpurun_out/c48/bench.err; echo "rc $?" >> gpurun_out/c48/bench.err
