#!/bin/bash
# session-4 call 20: PRE H1 loop unroll A/B (W0 loads in flight)
O=gpurun_out/s4c20
mkdir -p $O
export PYTHONUNBUFFERED=1
for v in default h1u5 h1u10 default h1u5 h1u10; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  echo "== $v" >> $O/trace.txt
  timeout 300 python tools/dec_trace.py --batches 1,16,24,40,64 --precision parity >> $O/trace.txt 2>&1
done
