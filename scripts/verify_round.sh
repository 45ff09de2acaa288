set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -6 > gpurun_out/v7_pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v7_smoke.txt 2>&1
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/v7_bench.json
cat gpurun_out/v7_pytest_gpu.txt gpurun_out/v7_smoke.txt gpurun_out/v7_bench.json
