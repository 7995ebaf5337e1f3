#!/bin/bash
# DEC_CONTIG=1 + projection-partial ILP: correctness, phase trace, ncu at B=24 / B=512
mkdir -p gpurun_out/c24
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py -q -rf -x > gpurun_out/c24/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c24/pytest.txt
timeout 300 python tools/dec_trace.py --batches 1,24,128,256,512 --precision parity > gpurun_out/c24/trace_parity.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dec_persist -s 1 -c 1 -o gpurun_out/c24/prof_dec24 python tools/dec_once.py 24 > gpurun_out/c24/ncu24.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dec_persist -s 1 -c 1 -o gpurun_out/c24/prof_dec512 python tools/dec_once.py 512 > gpurun_out/c24/ncu512.log 2>&1
