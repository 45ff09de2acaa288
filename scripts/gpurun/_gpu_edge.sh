mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -k "edge or config4 or unit or ieee or bench_step or single_rank" -q -s --timeout 900 2>&1 | tail -40 > gpurun_out/r02_edge.txt
cat gpurun_out/r02_edge.txt
