#!/bin/bash
# One multi-GPU lease answers every policy choice round 1 tuned on loopback:
#   bash scripts/nvlink_decisions.sh [N=8] [OUT=gpurun_out/decisions]
# plus the NCCL sweep (default and NVLS excluded) and the bench line at N.
# Dry run on one GPU: DDL_BENCH_SAME_GPU=1 bash scripts/nvlink_decisions.sh 2
set -x
N=${1:-8}
OUT=${OUT:-gpurun_out/decisions}
mkdir -p "$OUT"
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29651"
EXTRA=""
if [ "${DDL_BENCH_SAME_GPU:-0}" = "1" ]; then EXTRA="--iters 2 --max-bytes 4194304"; fi
# NVLink topology / P2P / multicast facts of this box
nvidia-smi topo -m > "$OUT/topo.txt" 2>&1
nvidia-smi nvlink -s > "$OUT/nvlink_status.txt" 2>&1
timeout 3000 $RUN scripts/nvlink_decisions.py --out-dir "$OUT" $EXTRA 2>&1 | tail -20 > "$OUT/decisions.log"
if [ "${DDL_BENCH_SAME_GPU:-0}" != "1" ]; then
  timeout 1800 $RUN scripts/sweep.py --config sweep --out "$OUT/sweep_nccl_P$N.csv" > "$OUT/sweep.log" 2>&1
  NCCL_NVLS_ENABLE=0 timeout 1800 $RUN scripts/sweep.py --config sweep --out "$OUT/sweep_nccl_nonvls_P$N.csv" \
    > "$OUT/sweep_nonvls.log" 2>&1
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 600 $RUN bench.py --gpus $N --steps 20 --warmup 5 \
    > "$OUT/bench_P$N.log" 2>&1
  OUT="$OUT/nvl" bash scripts/ncu_nvlink.sh $N > "$OUT/ncu_nvlink.log" 2>&1 || true
fi
ls -la "$OUT"
