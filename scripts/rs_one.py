"""One loopback reduce-scatter call (ncu target): P = 8, dims from argv (default 2x4),
recv elements from argv (default 1M fp32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl
spec = sys.argv[1] if len(sys.argv) > 1 else "2x4"
recv = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
lb = ddl.Loopback(8, ddl.parse_dims(spec))
sends = [torch.full((8 * recv,), float(r + 1), device="cuda") for r in range(8)]
outs = [torch.empty(recv, device="cuda") for _ in range(8)]
for _ in range(4):
    lb.reduce_scatter(outs, sends)
torch.cuda.synchronize()
assert all(bool((o == 36).all()) for o in outs)
