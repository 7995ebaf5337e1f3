#!/bin/bash
mkdir -p gpurun_out/c71
export PYTHONUNBUFFERED=1
for v in default cnoinl base default cnoinl base; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  timeout 300 python tools/dec_trace.py --batches 16,128,256 --precision parity >> gpurun_out/c71/trace_$v.txt 2>&1
done
