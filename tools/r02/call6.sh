mkdir -p gpurun_out/c6
for n in Gp AP; do
  for B in 5 84 120; do
    timeout 120 python tools/poison_probe2.py $n --B $B >> gpurun_out/c6/probe.txt 2>&1
    timeout 120 python tools/poison_probe2.py $n --B $B --value nan >> gpurun_out/c6/probe.txt 2>&1
  done
  timeout 120 python tools/poison_probe2.py $n --B 84 --steps-all 32 >> gpurun_out/c6/probe.txt 2>&1
done
