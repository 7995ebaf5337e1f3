#!/bin/bash
# session-4 call 4: TMEM-resident decoder-gate weights -- decoder tests, A/B phase trace vs DEC_WRES=0
mkdir -p gpurun_out/s4c4
export PYTHONUNBUFFERED=1
O=gpurun_out/s4c4
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py tests/test_gpu_parity_r.py -q -x > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for v in default nowres default nowres; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  echo "== $v" >> $O/trace.txt
  timeout 300 python tools/dec_trace.py --batches 1,8,16,24,64,128 --precision parity >> $O/trace.txt 2>&1
done
unset ITTS_LIB
timeout 300 python tools/dec_trace.py --batches 16,64 --precision bf16 > $O/trace_bf16.txt 2>&1
