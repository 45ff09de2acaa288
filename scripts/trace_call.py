"""Per-phase timeline of one loopback all-reduce (DDL_TRACE=1): for every barrier j, the
wait (after previous phase -> barrier passed) and the phase that follows it, as
median / max over all CTAs of all virtual ranks, in microseconds.
python scripts/trace_call.py --dims 2x4 --bytes 31502336"""
import argparse, os, sys
os.environ["DDL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1811_12174_b200 import ddl

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=8)
ap.add_argument("--dims", default="2x4")
ap.add_argument("--bytes", type=int, default=31502336)
ap.add_argument("--algo", type=int, default=1)
a = ap.parse_args()
dims = ddl.parse_dims(a.dims)
lb = ddl.Loopback(a.P, dims)
lb.set_algo(a.algo, 0)
n = a.bytes // 4
bufs = [torch.ones(n, device="cuda") for _ in range(a.P)]
for _ in range(5):
    lb.all_reduce(bufs, "avg")
torch.cuda.synchronize()
tr = lb.trace().astype(np.int64)
C = lb.ctas_for(n, "float32")
tr = tr[:, :C, :]
L = sum(1 for g in dims if g > 1)
t0 = tr[:, :, 0].min()
us = lambda x: x / 1e3
print(f"P={a.P} dims={a.dims} bytes={a.bytes} ctas/rank={C}  total {us(tr[:, :, 2 + 4 * L].max() - t0):.1f} us")
prev = tr[:, :, 1]
print(f"  launch skew (start spread) {us(tr[:, :, 0].max() - t0):.1f}")
names = [f"RS{d}" for d in range(L)] + [f"AG{d}" for d in reversed(range(L))]
for j in range(2 * L):
    b = tr[:, :, 2 + 2 * j]
    f = tr[:, :, 3 + 2 * j]
    w = b - prev
    ph = f - b
    print(f"  barrier {j:2d}: wait med {us(np.median(w)):6.1f} max {us(w.max()):6.1f} | {names[j]:4s} med {us(np.median(ph)):6.1f} max {us(ph.max()):6.1f} | phase end spread {us(f.max() - f.min()):6.1f}")
    prev = f
end = tr[:, :, 2 + 4 * L]
print(f"  end barrier: wait med {us(np.median(end - prev)):.1f} max {us((end - prev).max()):.1f}")
