mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r02_v0_smi.txt; cat MEASURED_PEAKS.json >> gpurun_out/r02_v0_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -6 > gpurun_out/r02_v0_pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_v0_smoke.txt 2>&1
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/r02_v0_bench.json
cat gpurun_out/r02_v0_pytest_gpu.txt gpurun_out/r02_v0_smoke.txt gpurun_out/r02_v0_bench.json
