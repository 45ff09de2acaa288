mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_ddp.py tests/test_bench_contract.py -q -m gpu --timeout 900 2>&1 | tail -15 > gpurun_out/r02_v1_tests.txt
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -3 > gpurun_out/r02_v1_bench.json
ncu --query-metrics 2>/dev/null | grep -i nvl > gpurun_out/r02_nvl_metrics.txt
cat gpurun_out/r02_v1_tests.txt gpurun_out/r02_v1_bench.json
