"""Is the per-CTA phase-time spread systematic (same SMs slow every call) or random?
Runs K traced calls of one size; prints per-call RS0 durations' spread and the correlation
of per-CTA durations between calls, and the mean duration grouped by SM id."""
import argparse, os, sys
os.environ["DDL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1811_12174_b200 import ddl
ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="2x4")
ap.add_argument("--bytes", type=int, default=31502336)
ap.add_argument("--calls", type=int, default=8)
a = ap.parse_args()
P = 8
lb = ddl.Loopback(P, ddl.parse_dims(a.dims))
n = a.bytes // 4
bufs = [torch.ones(n, device="cuda") for _ in range(P)]
C = lb.ctas_for(n, "float32")
durs, sms = [], None
for k in range(a.calls + 2):
    lb.all_reduce(bufs, "avg")
    tr = lb.trace().astype(np.int64)[:, :C, :]
    if k < 2:
        continue
    d = (tr[:, :, 3] - tr[:, :, 2]).ravel() / 1e3   # RS0 duration per CTA (us)
    durs.append(d)
    sms = tr[:, :, 127].ravel()
D = np.array(durs)
print("per-call RS0 min/med/max:", [(round(x.min(), 1), round(np.median(x), 1), round(x.max(), 1)) for x in D])
cc = np.corrcoef(D)
print("mean correlation of per-CTA RS0 time between calls:", round((cc.sum() - len(D)) / (len(D) ** 2 - len(D)), 3))
m = D.mean(axis=0)
order = np.argsort(m)
print("slowest CTAs (mean us, smid):", [(round(m[i], 1), int(sms[i])) for i in order[-10:]])
print("fastest CTAs (mean us, smid):", [(round(m[i], 1), int(sms[i])) for i in order[:10]])
# by SM id
by = {}
for i, s_ in enumerate(sms):
    by.setdefault(int(s_), []).append(m[i])
sm_means = sorted((np.mean(v), k) for k, v in by.items())
print("SM mean RS0 (lowest 8):", [(round(v, 1), k) for v, k in sm_means[:8]])
print("SM mean RS0 (highest 8):", [(round(v, 1), k) for v, k in sm_means[-8:]])
