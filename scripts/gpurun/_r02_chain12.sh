mkdir -p gpurun_out
O=gpurun_out/r02_chain12.txt
: > $O
timeout 300 python scripts/step_ab.py "DDL_LB_CHAIN=0" "" >> $O 2>&1
for v in s6 s6r0 s5 s8 s6row s4; do
  echo "== $v" >> $O
  DDL_LIB=$PWD/build_variants/libddl_$v.so timeout 300 python scripts/step_ab.py "" "" >> $O 2>&1
done
echo "== k5" >> $O
timeout 300 python scripts/k5_bench.py >> $O 2>&1
python - >> $O 2>&1 <<'PY'
import torch
a = torch.empty(818*1024*1024//4, device="cuda"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("torch copy 818 MB: best %.4f ms -> %.1f GB/s (r+w)" % (min(ts), 2 * a.numel() * 4 / min(ts) / 1e6))
PY
cat $O
