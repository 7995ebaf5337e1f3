mkdir -p gpurun_out/c16
timeout 900 python -m pytest tests/test_gpu_decoder_paths.py -q -rf > gpurun_out/c16/pytest.txt 2>&1; echo "rc $?" >> gpurun_out/c16/pytest.txt
timeout 600 python tools/r02/parity_probe.py --chars 50,200 --precision parity --oracle-encoder > gpurun_out/c16/probe_parity_orcenc.txt 2>&1
timeout 600 python tools/r02/parity_probe.py --chars 50,200 --precision bf16 --oracle-encoder > gpurun_out/c16/probe_bf16_orcenc.txt 2>&1
