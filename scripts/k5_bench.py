"""K5 local reduce/scale microbench: out = s * sum_{j<g} in_j, bytes (g+1)*n*w vs HBM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl
for g in (2, 4, 8):
    for mb in (16, 64, 256):
        n = (mb << 20) // 4
        ins = [torch.randn(n, device="cuda") for _ in range(g)]
        out = torch.empty(n, device="cuda")
        for _ in range(3):
            ddl.local_reduce(ins, out, 1.0 / g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            ddl.local_reduce(ins, out, 1.0 / g)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"g={g} {mb}MiB {ms*1e3:.1f}us {(g+1)*n*4/(ms*1e-3)/1e9:.0f} GB/s")
        del ins, out
