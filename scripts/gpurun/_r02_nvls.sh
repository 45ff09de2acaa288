mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nvls.py tests/test_gpu_multiproc.py -q -m gpu --timeout 600 2>&1 | tail -25 > gpurun_out/r02_nvls_tests.txt
cat gpurun_out/r02_nvls_tests.txt
