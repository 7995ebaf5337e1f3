#!/bin/bash
# PDL re-check now that the stale-shared-memory decoder bug is fixed
mkdir -p gpurun_out/c45
export PYTHONUNBUFFERED=1
for i in 1 2 3; do
  ITTS_PDL_MASK=31 timeout 600 python tools/race_check.py --iters 300 --heavy > gpurun_out/c45/pdl_$i.txt 2>&1
done
ITTS_NO_PDL=1 timeout 600 python tools/race_check.py --iters 300 --heavy --serial > gpurun_out/c45/serial.txt 2>&1
ITTS_PDL_MASK=31 timeout 300 python tools/module_times.py --batches 16,128 > gpurun_out/c45/times_pdl.txt 2>&1
timeout 300 python tools/module_times.py --batches 16,128 > gpurun_out/c45/times_nopdl.txt 2>&1
