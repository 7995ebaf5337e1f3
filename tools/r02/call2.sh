#!/bin/bash
mkdir -p gpurun_out/c2
export PYTHONUNBUFFERED=1
export ITTS_LIB=$PWD/tools/bin/nomerge.so
timeout 420 python tools/soak.py --qps 200 --seconds 30 --diag-rerun --bisect-dir gpurun_out/c2/cases --no-graphs > gpurun_out/c2/soak_nomerge_bisect.txt 2>&1; echo "rc $?" >> gpurun_out/c2/soak_nomerge_bisect.txt
for c in gpurun_out/c2/cases/*.npz; do
  [ -f "$c" ] || continue
  ITTS_LIB=$PWD/tools/bin/nomerge.so timeout 200 python tools/dec_case.py $c --repeat 3 --solo > $c.nomerge.txt 2>&1
  unset ITTS_LIB; timeout 200 python tools/dec_case.py $c --repeat 3 --solo > $c.default.txt 2>&1
  timeout 200 python tools/dec_case.py $c --repeat 3 --graphs > $c.default_graphs.txt 2>&1
  break
done
unset ITTS_LIB
timeout 600 python tools/r02/parity_probe.py --chars 50,200,1000 > gpurun_out/c2/parity_probe.txt 2>&1
