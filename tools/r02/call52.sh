#!/bin/bash
mkdir -p gpurun_out/c52
export PYTHONUNBUFFERED=1
# stage-1 / stage-2 layer shapes at pooled batch 16 (rows ~ 16 x 36 x 8 + halos = 5400; x 8 = 37000)
for k in 3 11; do
timeout 120 python tools/rb_trace.py --rows 5400 --c 256 --k $k --dil 5 >> gpurun_out/c52/rb.txt 2>&1
timeout 120 python tools/rb_trace.py --rows 37000 --c 128 --k $k --dil 5 >> gpurun_out/c52/rb.txt 2>&1
timeout 120 python tools/rb_trace.py --rows 150000 --c 32 --k $k --dil 5 >> gpurun_out/c52/rb.txt 2>&1
done
