#!/bin/bash
# Round 2, call 1: GPU test suite + soak A/B on the intermittent non-finite chunks.
mkdir -p gpurun_out/c1
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/c1/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/c1/pytest_gpu.txt
for v in "eager_default:--no-graphs:" "eager_nomerge:--no-graphs:tools/bin/nomerge.so" "graph_default::" "eager_default2:--no-graphs:"; do
  name=${v%%:*}; rest=${v#*:}; flags=${rest%%:*}; lib=${rest#*:}
  if [ -n "$lib" ]; then export ITTS_LIB=$PWD/$lib; else unset ITTS_LIB; fi
  timeout 300 python tools/soak.py --qps 200 --seconds 30 --diag-rerun $flags > gpurun_out/c1/soak_$name.txt 2>&1
  echo "rc $?" >> gpurun_out/c1/soak_$name.txt
done
unset ITTS_LIB
