#!/bin/bash
mkdir -p gpurun_out/c74
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py tests/test_gpu_parity_r.py -q -x > gpurun_out/c74/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c74/pytest.txt
for v in default prev default prev; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  timeout 300 python tools/dec_trace.py --batches 1,8,16,20,24,32 --precision parity >> gpurun_out/c74/trace_$v.txt 2>&1
done
