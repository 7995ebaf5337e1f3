#!/bin/bash
mkdir -p gpurun_out/c50
export PYTHONUNBUFFERED=1
# k_conv_tc launches of one vocoder call at B=230: conv_pre, convT1..3 (BN 128), convT4 (BN 64)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 4 -c 6 -o gpurun_out/c50/convs python tools/profile_iter.py --batches 230 --iters 1 > gpurun_out/c50/ncu.log 2>&1
