#!/bin/bash
# session-4 call 13: same-box A/B of the C3 headline (100 QPS, 30 s) -- barrier-free attention schedule vs DEC_ITEM_CNT=0
O=gpurun_out/s4c13
mkdir -p $O
export PYTHONUNBUFFERED=1
for v in default noicnt default noicnt default noicnt; do
  if [ $v = default ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --sweep "" --side-configs 0 --no-cpu-baseline > $O/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1])
print('$v', 'p99', d['value'], 'p50', d['p50_ms'], 'e2e', d['e2e']['value'], 'thirds', d['p99_ms_by_third_of_window'], 'dec', d['module_device_ms_per_iteration'], 'B', d['pooled_batch_mean'])" >> $O/ab.txt
done
