#!/bin/bash
# session-4 final validation: GPU suite, smoke, bench (ours + reference arm), 13 soaks at 200 QPS,
# ncu launch lists + full captures (tools/profile_round.sh)
O=gpurun_out/s4f
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/ -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc $?" >> $O/smoke.txt
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc $?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc $?" >> $O/bench_ref.err
for i in 1 2 3 4 5 6 7 8 9 10; do
  echo "== soak graph $i" >> $O/soak.txt
  timeout 240 python tools/soak.py --qps 200 --seconds 60 2>&1 | grep -E "inside the timed|requests |engine failure|diag" >> $O/soak.txt
done
for i in 1 2 3; do
  echo "== soak eager $i" >> $O/soak.txt
  timeout 240 python tools/soak.py --qps 200 --seconds 60 --no-graphs 2>&1 | grep -E "inside the timed|requests |engine failure|diag" >> $O/soak.txt
done
bash tools/profile_round.sh > $O/profile_round.log 2>&1
