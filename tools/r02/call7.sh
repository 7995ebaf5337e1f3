mkdir -p gpurun_out/c7
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool initcheck --print-limit 30 python tools/r02/san_case.py 84 4 > gpurun_out/c7/initcheck.txt 2>&1; echo "rc $?" >> gpurun_out/c7/initcheck.txt
timeout 900 $CS --tool memcheck --print-limit 30 python tools/r02/san_case.py 84 4 > gpurun_out/c7/memcheck.txt 2>&1; echo "rc $?" >> gpurun_out/c7/memcheck.txt
timeout 1200 $CS --tool racecheck --racecheck-report hazard --print-limit 30 python tools/r02/san_case.py 84 2 > gpurun_out/c7/racecheck.txt 2>&1; echo "rc $?" >> gpurun_out/c7/racecheck.txt
