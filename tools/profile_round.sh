#!/bin/bash
# GPU-side profiling pass for one round (run under gpurun).  Outputs in gpurun_out/:
#   launches_b128.csv   ncu launch list (gpu__time_duration.sum) of one decoder + vocoder call at B=128
#   prof_conv.ncu-rep   ncu --set full: 2 stage-2 HiFi-GAN MRF convs (k=3 c1, k=3 c2 +residual)
#   prof_attn.ncu-rep   ncu --set full: the attention kernel (4-CTA clusters)
#   prof_gemm.ncu-rep   ncu --set full: a decoder gate GEMM (K-split)
# (ncu on bench.py itself distorts the serving dynamics -- the pool grows while kernels are
#  serialised -- so the launch list is taken on the fixed-batch profile_iter workload.)
P="python tools/profile_iter.py --batches 128 --iters 1 --no-graphs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b128.csv $P > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 89 -c 2 -o gpurun_out/prof_conv $P > gpurun_out/ncu_conv.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attention -s 5 -c 1 -o gpurun_out/prof_attn $P > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 6 -c 1 -o gpurun_out/prof_gemm $P > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out
