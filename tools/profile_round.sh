#!/bin/bash
# GPU-side profiling pass (run under gpurun).  Outputs in gpurun_out/:
#   launches_b24.csv / launches_b128.csv   ncu launch lists (gpu__time_duration.sum) of one decoder +
#                                          vocoder call at pooled batch 24 (~100 QPS) and 128 (~175 QPS)
#   prof_dec24.ncu-rep                     ncu --set full: the persistent decoder-chunk kernel, B=24
#   prof_rb_c128.ncu-rep / prof_rb_c32     ncu --set full: fused ResBlock layers (stage 2 k=7, stage 4 k=11), B=24
set -x
P24="python tools/profile_iter.py --batches 24 --iters 2"
P128="python tools/profile_iter.py --batches 128 --iters 2"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b24.csv $P24 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b128.csv $P128 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dec_persist -s 1 -c 1 -o gpurun_out/prof_dec24 python tools/dec_once.py 24 > gpurun_out/ncu_dec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 12 -c 1 -o gpurun_out/prof_rb_c128 $P24 > gpurun_out/ncu_rb.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 35 -c 1 -o gpurun_out/prof_rb_c32 $P24 > gpurun_out/ncu_rb2.log 2>&1
ls -la gpurun_out
