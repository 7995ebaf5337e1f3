#!/bin/bash
# session-4 call 5: PRE weights in smem + TMEM-resident gate weights (A/B variants)
mkdir -p gpurun_out/s4c5
export PYTHONUNBUFFERED=1
O=gpurun_out/s4c5
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py tests/test_gpu_parity_r.py -q -x > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for v in default wres1 nowres base default wres1 nowres base; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  echo "== $v" >> $O/trace.txt
  timeout 300 python tools/dec_trace.py --batches 1,8,16,24,40,64 --precision parity >> $O/trace.txt 2>&1
done
