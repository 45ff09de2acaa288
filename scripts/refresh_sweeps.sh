# Configs 3-5 on the current build (loopback, CUDA-graph timed, closed-form gated): one CSV each.
mkdir -p gpurun_out
TAG=${TAG:-r02}
rm -f gpurun_out/${TAG}_loopback_sweep.csv gpurun_out/${TAG}_loopback_bf16.csv gpurun_out/${TAG}_loopback_unet3d.csv
timeout 900 python scripts/sweep.py --config sweep --out gpurun_out/${TAG}_loopback_sweep.csv > gpurun_out/${TAG}_sweep_sweep.log 2>&1
timeout 900 python scripts/sweep.py --config bf16 --out gpurun_out/${TAG}_loopback_bf16.csv > gpurun_out/${TAG}_sweep_bf16.log 2>&1
timeout 900 python scripts/sweep.py --config unet3d --out gpurun_out/${TAG}_loopback_unet3d.csv > gpurun_out/${TAG}_sweep_unet3d.log 2>&1
tail -3 gpurun_out/${TAG}_loopback_*.csv
