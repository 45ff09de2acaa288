mkdir -p gpurun_out
bash scripts/gpu_mutation_check.sh > gpurun_out/r02_gpu_mutations2.txt 2>&1
cat gpurun_out/r02_gpu_mutations2.txt
TAG=r02d bash scripts/refresh_sweeps.sh > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_grouped.py tests/test_gpu_ll.py -q --timeout 1400 2>&1 | tail -3 > gpurun_out/r02_mut_tests.txt
cat gpurun_out/r02_mut_tests.txt
cat gpurun_out/r02d_loopback_unet3d.csv gpurun_out/r02d_loopback_bf16.csv
