#!/bin/bash
mkdir -p gpurun_out/c3; rm -rf /tmp/c3cases
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_decoder_paths.py -q -rA > gpurun_out/c3/pytest_dec.txt 2>&1; echo "rc $?" >> gpurun_out/c3/pytest_dec.txt
for i in 1 2 3; do
 for v in "default:" "nomerge:tools/bin/nomerge.so"; do
  name=${v%%:*}; lib=${v#*:}
  if [ -n "$lib" ]; then export ITTS_LIB=$PWD/$lib; else unset ITTS_LIB; fi
  timeout 400 python tools/soak.py --qps 200 --seconds 30 --diag-rerun --bisect-dir /tmp/c3cases/${name}_$i --no-graphs > gpurun_out/c3/soak_${name}_$i.txt 2>&1
  echo "rc $?" >> gpurun_out/c3/soak_${name}_$i.txt
 done
done
unset ITTS_LIB
for c in /tmp/c3cases/*/*.npz; do
  [ -f "$c" ] || continue
  timeout 200 python tools/dec_case.py $c --repeat 3 --solo > gpurun_out/c3/$(basename $(dirname $c))_$(basename $c).default.txt 2>&1
  ITTS_LIB=$PWD/tools/bin/nomerge.so timeout 200 python tools/dec_case.py $c --repeat 3 > gpurun_out/c3/$(basename $(dirname $c))_$(basename $c).nomerge.txt 2>&1
done
