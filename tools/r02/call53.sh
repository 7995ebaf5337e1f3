#!/bin/bash
mkdir -p gpurun_out/c53
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/c53/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c53/pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c53/smoke.txt 2>&1; echo "rc $?" >> gpurun_out/c53/smoke.txt
timeout 300 python tools/dec_trace.py --batches 1,16,24,128,256,512 --precision parity > gpurun_out/c53/trace.txt 2>&1
timeout 1800 python bench.py > gpurun_out/c53/bench.txt 2>gpurun_out/c53/bench.err; echo "rc $?" >> gpurun_out/c53/bench.err
timeout 1200 bash tools/profile_round.sh > gpurun_out/c53/profile.log 2>&1
