#!/bin/bash
# Vocoder profiling pass (run under gpurun): launch list of one B=128 decoder+vocoder call and
# ncu --set full captures of fused ResBlock layers of the native launch sequence (per stage:
# branch 0, 1, 2 x 3 layers; stage 3 = C 64: launches 18..26, stage 4 = C 32: 27..35).
P="python tools/profile_iter.py --batches 128 --iters 1 --no-graphs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_voc2.csv $P > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 33 -c 1 -o gpurun_out/prof_rb_c32_k11 $P > gpurun_out/ncu_rb_c32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 24 -c 1 -o gpurun_out/prof_rb_c64_k11 $P > gpurun_out/ncu_rb_c64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 6 -c 1 -o gpurun_out/prof_rb_c256_k11 $P > gpurun_out/ncu_rb_c256.log 2>&1
ls -la gpurun_out | tail -5
