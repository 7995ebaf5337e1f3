mkdir -p gpurun_out/c9
for n in Gp AP; do for L in 1 2; do
timeout 120 python tools/poison_probe3.py $n --B 84 --left $L >> gpurun_out/c9/p3.txt 2>&1
done; done
timeout 120 python tools/poison_probe3.py Gp --B 84 --left 1 --value 12345 >> gpurun_out/c9/p3.txt 2>&1
for v in clobber wfence nomerge; do
  echo "== variant $v" >> gpurun_out/c9/p3.txt
  ITTS_LIB=$PWD/tools/bin/$v.so timeout 120 python tools/poison_probe3.py Gp --B 84 --left 1 >> gpurun_out/c9/p3.txt 2>&1
done
