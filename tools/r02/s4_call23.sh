#!/bin/bash
# session-4 call 23: ATT-A context loop unrolled 8
O=gpurun_out/s4c23
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py tests/test_gpu_parity_r.py tests/test_gpu_tier_r.py -q -x > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
for v in default prevctx default prevctx; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  echo "== $v" >> $O/trace.txt
  timeout 300 python tools/dec_trace.py --batches 16,24,128,256 --precision parity >> $O/trace.txt 2>&1
done
unset ITTS_LIB
timeout 300 python tools/race_check.py --heavy --iters 200 > $O/race.txt 2>&1
timeout 300 python tools/race_check.py --heavy --iters 200 --no-graphs >> $O/race.txt 2>&1
