#!/bin/bash
# session-4 final re-validation (decoder PRE / combine load batching): GPU suite, smoke, bench, reference arm, 7 soaks, ncu at B=16
O=gpurun_out/s4f3
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/ -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc $?" >> $O/smoke.txt
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc $?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc $?" >> $O/bench_ref.err
for i in 1 2 3 4 5; do
  echo "== soak graph $i" >> $O/soak.txt
  timeout 240 python tools/soak.py --qps 200 --seconds 60 2>&1 | grep -E "inside the timed|requests |engine failure|diag" >> $O/soak.txt
done
for i in 1 2; do
  echo "== soak eager $i" >> $O/soak.txt
  timeout 240 python tools/soak.py --qps 200 --seconds 60 --no-graphs 2>&1 | grep -E "inside the timed|requests |engine failure|diag" >> $O/soak.txt
done
P16="python tools/profile_iter.py --batches 16 --iters 2"; mkdir -p gpurun_out/prof3; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof3/launches_b16.csv $P16 > /dev/null 2>&1; timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dec_persist -s 1 -c 1 -o gpurun_out/prof3/dec16 python tools/dec_once.py 16 > gpurun_out/prof3/ncu_dec16.log 2>&1
