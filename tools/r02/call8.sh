mkdir -p gpurun_out/c8
CS="/usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5"
for v in base clobber wfence nomerge; do
  if [ $v = base ]; then unset ITTS_LIB; else export ITTS_LIB=$PWD/tools/bin/$v.so; fi
  for B in 84 5; do
    echo "== $v B=$B" >> gpurun_out/c8/res.txt
    timeout 300 $CS python tools/r02/san_case.py $B 4 2>&1 | grep -E "finite|ERROR SUMMARY" >> gpurun_out/c8/res.txt
  done
done
