#!/bin/bash
# round-2 session-3 first call: full GPU suite, default bench, soaks with default GC, launch lists
mkdir -p gpurun_out/c21
export PYTHONUNBUFFERED=1
nvidia-smi > gpurun_out/c21/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/c21/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c21/pytest.txt
timeout 900 python bench.py > gpurun_out/c21/bench.txt 2>gpurun_out/c21/bench.err; echo "rc $?" >> gpurun_out/c21/bench.err
for i in 1 2 3; do
  timeout 300 python tools/soak.py --qps 200 --seconds 60 > gpurun_out/c21/soak_$i.txt 2>&1; echo "rc $?" >> gpurun_out/c21/soak_$i.txt
done
timeout 900 bash tools/profile_round.sh > gpurun_out/c21/profile.log 2>&1
