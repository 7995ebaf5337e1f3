mkdir -p gpurun_out/c15
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py tests/test_gpu_parity_r.py tests/test_gpu_tier_r.py -q -rf -s > gpurun_out/c15/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c15/pytest.txt
for p in parity bf16; do
  timeout 600 python tools/r02/parity_probe.py --chars 50,200,1000 --precision $p > gpurun_out/c15/probe_$p.txt 2>&1
  timeout 300 python tools/dec_trace.py --batches 1,24,128,256 --precision $p > gpurun_out/c15/trace_$p.txt 2>&1
done
