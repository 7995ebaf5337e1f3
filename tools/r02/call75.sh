#!/bin/bash
mkdir -p gpurun_out/c75
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_tier_r.py tests/test_gpu_resblock.py tests/test_gpu_parity_r.py -q -x > gpurun_out/c75/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c75/pytest.txt
for v in default prevlib default prevlib; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  timeout 300 python tools/module_times.py --batches 8,16,32,128 --reps 30 >> gpurun_out/c75/mt_$v.txt 2>&1
done
