"""Per-channel timeline of one grouped all-reduce of the bench step (DDL_TRACE=1): for every
bucket-wave k and phase j of each channel, the barrier wait and the phase duration (median /
max over that channel's CTAs of all virtual ranks, microseconds), and when each channel ends.
  python scripts/trace_grouped.py [--dims 2x4]"""
import argparse
import os
import sys

os.environ["DDL_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_12174_b200 import ddl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="2x4")
a = ap.parse_args()
P, dims = 8, ddl.parse_dims(a.dims)
L = sum(1 for g in dims if g > 1)
lb = ddl.Loopback(P, dims)
host = [bench.resnet50_set(r) for r in range(P)]
bufs = [[torch.from_numpy(host[r][b]).cuda() for r in range(P)] for b in range(len(host[0]))]
for _ in range(6):
    lb.all_reduce_many(bufs, "avg")
torch.cuda.synchronize()
tr = lb.trace().astype(np.int64)          # [P][cmax][128]
C = 37
tr = tr[:, :C, :]
t0 = tr[:, :, 0].min()
us = lambda x: x / 1e3                    # noqa: E731
nev = (tr[:, :, 1:127] > 0).sum(axis=2)    # events recorded per CTA -> its channel's bucket-waves
end_ev = [tr[r, c, 1:127][tr[r, c, 1:127] > 0].max() for r in range(P) for c in range(C)]
print(f"grouped step, dims {a.dims}: total {us(max(end_ev) - t0):.1f} us")
for ne in sorted(set(nev.ravel().tolist())):
    sel = nev == ne
    nk = ne // (4 * L)
    ctas = sorted(set(np.nonzero(sel)[1].tolist()))
    print(f"channel with {nk} bucket(s), CTAs {ctas[0]}..{ctas[-1]}:")
    prev = tr[:, :, 0][sel]
    for k in range(nk):
        for j in range(2 * L):
            b = tr[:, :, 1 + 2 * (k * 2 * L + j)][sel]
            f = tr[:, :, 2 + 2 * (k * 2 * L + j)][sel]
            name = f"RS{j}" if j < L else f"AG{2 * L - 1 - j}"
            print(f"  bucket {k} {name:4s}: wait med {us(np.median(b - prev)):6.1f} max {us((b - prev).max()):6.1f}"
                  f" | phase med {us(np.median(f - b)):6.1f} max {us((f - b).max()):6.1f}"
                  f" | ends {us(np.median(f - t0)):6.1f}..{us(f.max() - t0):6.1f}")
            prev = f
lb.finalize()
