#!/bin/bash
# GPU-side profiling pass (run under gpurun).  Outputs in gpurun_out/prof/:
#   launches_b16.csv / launches_b230.csv   ncu launch lists (gpu__time_duration.sum) of serving iterations
#                                          at pooled batch 16 (~100 QPS) and 230 (~300 QPS)
#   dec16.ncu-rep / dec230.ncu-rep         ncu --set full: the persistent decoder-chunk kernel
#   rb_c128.ncu-rep / rb_c32.ncu-rep       ncu --set full: fused ResBlock layers (stage 2 k=7, stage 4 k=11), B=16
set -x
mkdir -p gpurun_out/prof
P16="python tools/profile_iter.py --batches 16 --iters 2"
P230="python tools/profile_iter.py --batches 230 --iters 2"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_b16.csv $P16 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_b230.csv $P230 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dec_persist -s 1 -c 1 -o gpurun_out/prof/dec16 python tools/dec_once.py 16 > gpurun_out/prof/ncu_dec16.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dec_persist -s 1 -c 1 -o gpurun_out/prof/dec230 python tools/dec_once.py 230 > gpurun_out/prof/ncu_dec230.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 12 -c 1 -o gpurun_out/prof/rb_c128 $P16 > gpurun_out/prof/ncu_rb.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 35 -c 1 -o gpurun_out/prof/rb_c32 $P16 > gpurun_out/prof/ncu_rb2.log 2>&1
ls -la gpurun_out/prof
