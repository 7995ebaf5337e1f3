#!/bin/bash
# session-4 last check of the committed head: GPU suite, smoke, full bench
O=gpurun_out/s4f4
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/ -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc $?" >> $O/smoke.txt
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc $?" >> $O/bench.err
