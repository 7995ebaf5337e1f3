#!/bin/bash
mkdir -p gpurun_out/c67
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c67/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c67/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c67/smoke.txt 2>&1; echo "rc $?" >> gpurun_out/c67/smoke.txt
timeout 1800 python bench.py > gpurun_out/c67/bench.txt 2>gpurun_out/c67/bench.err; echo "rc $?" >> gpurun_out/c67/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/c67/bench_ref.txt 2>gpurun_out/c67/bench_ref.err; echo "rc $?" >> gpurun_out/c67/bench_ref.err
bash tools/profile_round.sh > gpurun_out/c67/prof.log 2>&1
