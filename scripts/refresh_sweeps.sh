mkdir -p gpurun_out
timeout 900 python scripts/sweep.py --config sweep --out gpurun_out/r01_loopback_sweep.csv > gpurun_out/sweep_sweep.log 2>&1
timeout 900 python scripts/sweep.py --config bf16 --out gpurun_out/r01_loopback_bf16.csv > gpurun_out/sweep_bf16.log 2>&1
timeout 900 python scripts/sweep.py --config unet3d --out gpurun_out/r01_loopback_unet3d.csv > gpurun_out/sweep_unet3d.log 2>&1
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/v11_bench.json
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -4 > gpurun_out/v11_pytest_gpu.txt
cat gpurun_out/v11_pytest_gpu.txt
