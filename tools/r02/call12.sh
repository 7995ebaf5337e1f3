mkdir -p gpurun_out/c12
timeout 600 python -m pytest tests/test_gpu_decoder_paths.py -q -rA > gpurun_out/c12/pytest_dec.txt 2>&1; echo "rc $?" >> gpurun_out/c12/pytest_dec.txt
timeout 120 python tools/poison_probe4.py Gp > gpurun_out/c12/p4.txt 2>&1
for i in 1 2; do
  timeout 400 python tools/soak.py --qps 200 --seconds 30 --diag-rerun --no-graphs > gpurun_out/c12/soak_eager_$i.txt 2>&1; echo "rc $?" >> gpurun_out/c12/soak_eager_$i.txt
  timeout 400 python tools/soak.py --qps 200 --seconds 30 --diag-rerun > gpurun_out/c12/soak_graph_$i.txt 2>&1; echo "rc $?" >> gpurun_out/c12/soak_graph_$i.txt
done
