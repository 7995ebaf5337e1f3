#!/bin/bash
# session-4 call 2: vocoder poison test, decoder phase trace, module times
mkdir -p gpurun_out/s4c2
export PYTHONUNBUFFERED=1
O=gpurun_out/s4c2
timeout 600 python -m pytest tests/test_gpu_tier_r.py -q -x -k "poison or unwritten or batched_vocoder" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 300 python tools/dec_trace.py --batches 1,8,16,24,64,128 --precision parity > $O/trace.txt 2>&1
timeout 300 python tools/module_times.py --batches 8,16,32,128 --reps 30 > $O/mt.txt 2>&1
