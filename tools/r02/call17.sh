mkdir -p gpurun_out/c17
for p in parity bf16; do
timeout 600 python tools/r02/parity_probe.py --chars 50,200,1000 --precision $p > gpurun_out/c17/probe_$p.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_tier_r.py tests/test_gpu_parity_r.py -q -rf > gpurun_out/c17/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c17/pytest.txt
