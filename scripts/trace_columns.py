import os, sys
os.environ["DDL_TRACE"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1811_12174_b200 import ddl
P = 8
lb = ddl.Loopback(P, [4, 2])
n = 31502336 // 4
bufs = [torch.ones(n, device="cuda") for _ in range(P)]
C = lb.ctas_for(n, "float32")
for k in range(6):
    lb.all_reduce(bufs, "avg")
    tr = lb.trace().astype(np.int64)[:, :C, :]
    if k < 2: continue
    t0 = tr[:, :, 0].min()
    L = 2
    end_phase = [tr[:, :, 3 + 2 * j] - t0 for j in range(2 * L)]  # [P, C]
    col_end = [e.max(axis=0) for e in end_phase]                  # per column
    print("call", k, "phase-end: col-max spread (us):", [round((c.max() - c.min()) / 1e3, 1) for c in col_end],
          " all-CTA spread:", [round((e.max() - e.min()) / 1e3, 1) for e in end_phase],
          " total:", round((tr[:, :, 2 + 4 * L].max() - t0) / 1e3, 1))
