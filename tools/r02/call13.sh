mkdir -p gpurun_out/c13
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/c13/pytest_gpu.txt 2>&1; echo "rc $?" >> gpurun_out/c13/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c13/smoke.txt 2>&1; echo "rc $?" >> gpurun_out/c13/smoke.txt
