"""One K5 local reduce (the bench.py `local_reduce` object: g = 8 inputs, 64 MiB fp32 output,
x 1/8) after W warm-ups -- the target of the K5 ncu capture:
  ncu --set full -k regex:local_reduce -s W -c 1 python scripts/profile_k5.py --warmup W"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl

ap = argparse.ArgumentParser()
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--g", type=int, default=8)
ap.add_argument("--mib", type=int, default=64)
a = ap.parse_args()
n = (a.mib << 20) // 4
ins = [torch.randn(n, device="cuda") for _ in range(a.g)]
out = torch.empty(n, device="cuda")
for _ in range(a.warmup + 1):
    ddl.local_reduce(ins, out, 1.0 / a.g)
torch.cuda.synchronize()
print("k5", a.g, a.mib, "MiB out, algorithmic bytes", (a.g + 1) * n * 4)
