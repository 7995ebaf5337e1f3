#!/bin/bash
mkdir -p gpurun_out/c60
export PYTHONUNBUFFERED=1
for v in default merge160 merge48; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  timeout 300 python tools/dec_trace.py --batches 16,48,64,96,128,160 --precision parity > gpurun_out/c60/trace_$v.txt 2>&1
done
