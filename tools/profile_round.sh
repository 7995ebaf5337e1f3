#!/bin/bash
# GPU-side profiling pass for one round (run under gpurun).  Produces in gpurun_out/:
#   launches_bench.csv   ncu launch list (gpu__time_duration.sum) of a short bench run
#   prof_conv.ncu-rep    ncu --set full of 2 HiFi-GAN conv launches (stage-2 MRF)
#   prof_attn.ncu-rep    ncu --set full of the attention kernel
#   prof_gemm.ncu-rep    ncu --set full of a decoder gate GEMM
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 20 --warmup 3 --warmup-seconds 2 --drain-seconds 1 --no-cpu-baseline --sweep "" \
  > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 155 -c 2 \
  -o gpurun_out/prof_conv python tools/profile_iter.py --batches 128 --iters 1 > gpurun_out/ncu_conv.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attention -s 5 -c 1 \
  -o gpurun_out/prof_attn python tools/profile_iter.py --batches 128 --iters 1 > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 6 -c 1 \
  -o gpurun_out/prof_gemm python tools/profile_iter.py --batches 128 --iters 1 > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out
