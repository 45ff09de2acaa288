#!/bin/bash
# NVLink evidence of SURVEY 8(d) for the N > 1 bench step: per-rank NVLink TX/RX bytes
# (user data vs all, i.e. protocol overhead), DRAM bytes and kernel time of the grouped
# all-reduce, one ncu report per rank.
#   bash scripts/ncu_nvlink.sh [N=8] [OUT=gpurun_out/nvl]
# Kernel replay would re-run one rank's kernel alone and its device barriers would never
# complete, so every rank is profiled with --replay-mode application and a metric list that
# fits one pass (SURVEY 8(d) "ncu with cross-GPU spinning kernels").  Metric names checked
# against `ncu --query-metrics` on the B200 (profiles/r02_ncu_nvlink_metric_names.txt).
set -x
N=${1:-8}
OUT=${OUT:-gpurun_out/nvl}
mkdir -p "$(dirname "$OUT")"
M=nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
  --master-port 29661 --no-python \
  ncu --replay-mode application --app-replay-buffer memory --clock-control none --metrics "$M" \
      -k regex:ddl_multi -s 5 -c 2 -f -o "${OUT}_rank%q{RANK}" \
      python bench.py --gpus "$N" --steps 3 --warmup 5 --no-cpu-baseline > "${OUT}.log" 2>&1
for r in $(seq 0 $((N - 1))); do
  ncu -i "${OUT}_rank${r}.ncu-rep" --page raw --csv --metrics "$M" > "${OUT}_rank${r}.csv" 2>/dev/null
done
ls -la "$(dirname "$OUT")"
