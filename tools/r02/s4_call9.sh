#!/bin/bash
# session-4 call 9: ATT-A memory rows on their own mbarrier (energies start after the pm rows)
mkdir -p gpurun_out/s4c9
export PYTHONUNBUFFERED=1
O=gpurun_out/s4c9
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py tests/test_gpu_parity_r.py -q -x > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for v in default prev default prev; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  echo "== $v" >> $O/trace.txt
  timeout 300 python tools/dec_trace.py --batches 1,16,24,64,128,256 --precision parity >> $O/trace.txt 2>&1
done
