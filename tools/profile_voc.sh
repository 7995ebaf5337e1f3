#!/bin/bash
# Vocoder profiling pass (run under gpurun): launch list of one B=128 decoder+vocoder call and
# ncu --set full captures of fused ResBlock layers (stage 2 = C 128: launches 9..17).
P="python tools/profile_iter.py --batches 128 --iters 1 --no-graphs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_voc.csv $P > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 9 -c 2 -o gpurun_out/prof_rb_k3 $P > gpurun_out/ncu_rb1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 15 -c 1 -o gpurun_out/prof_rb_k11 $P > gpurun_out/ncu_rb2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resblock_tc -s 0 -c 1 -o gpurun_out/prof_rb_c256 $P > gpurun_out/ncu_rb3.log 2>&1
ls -la gpurun_out
