#!/bin/bash
# session-4 call 1: full GPU suite, smoke, compute-sanitizer over a short serving replay
mkdir -p gpurun_out/s4c1
export PYTHONUNBUFFERED=1
O=gpurun_out/s4c1
timeout 1500 python -m pytest tests/ -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc $?" >> $O/smoke.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python tools/race_check.py --no-graphs --iters 10 > $O/san_$tool.txt 2>&1; echo "rc $?" >> $O/san_$tool.txt
done
timeout 1200 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python tools/race_check.py --no-graphs --iters 4 > $O/san_racecheck.txt 2>&1; echo "rc $?" >> $O/san_racecheck.txt
