"""Where the bench step's time goes (DDL_TRACE=1, loopback grouped all-reduce of the
ResNet-50 set, 8 virtual ranks): per channel the summed median phase and barrier-wait times,
each CTA's busy (in-phase) share of the step, and whether slow CTAs are tied to SMs.
  DDL_...=... python scripts/trace_step.py [--dims 2x4] [--calls 3]"""
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
ap.add_argument("--calls", type=int, default=3)
a = ap.parse_args()
P, dims = 8, ddl.parse_dims(a.dims)
L = sum(1 for g in dims if g > 1)
lb = ddl.Loopback(P, dims)
host = [bench.resnet50_set(r) for r in range(P)]
bufs = [[torch.from_numpy(host[r][b]).cuda() for r in range(P)] for b in range(len(host[0]))]
C = lb.ctas_for(1 << 30, "float32")   # upper bound; trimmed below to CTAs that recorded events
busy_runs = []
for call in range(5 + a.calls):
    lb.all_reduce_many(bufs, "avg")
    torch.cuda.synchronize()
    if call < 5:
        continue
    tr = lb.trace().astype(np.int64)
    sm = tr[:, :, 127]
    ev = tr[:, :, 1:127]
    used = (ev > 0).any(axis=2).any(axis=0)
    ncta = int(used.sum())
    tr, sm, ev = tr[:, :ncta], sm[:, :ncta], ev[:, :ncta]
    t0 = tr[:, :, 0].min()
    end = np.where(ev > 0, ev, 0).max(axis=2)
    total = (end.max() - t0) / 1e3
    # events: 1 + 2*(seq*2L + j) after barrier j of bucket-wave seq, +1 after its phase
    nev = (ev > 0).sum(axis=2)
    busy = np.zeros((P, ncta))
    wait = np.zeros((P, ncta))
    for r in range(P):
        for c in range(ncta):
            e = tr[r, c, 1:1 + nev[r, c]]
            prev = tr[r, c, 0]
            for i in range(0, len(e) - 1, 2):
                wait[r, c] += e[i] - prev
                busy[r, c] += e[i + 1] - e[i]
                prev = e[i + 1]
    busy_runs.append(busy)
    print(f"call {call}: step {total:.1f} us over {ncta} CTAs/rank; median busy {np.median(busy) / 1e3:.1f} us, "
          f"median wait {np.median(wait) / 1e3:.1f} us, busy share {np.sum(busy) / (P * ncta * total * 1e3):.3f}")
    # channel split: CTAs with the same event count belong to one channel
    for ne in sorted(set(nev[0].tolist())):
        cs = np.nonzero(nev[0] == ne)[0]
        print(f"  channel of {ne // (4 * L) if L else 0} bucket-waves, CTAs {cs[0]}..{cs[-1]}: busy med "
              f"{np.median(busy[:, cs]) / 1e3:.1f} us (min {busy[:, cs].min() / 1e3:.1f} max {busy[:, cs].max() / 1e3:.1f}), "
              f"wait med {np.median(wait[:, cs]) / 1e3:.1f} us, ends {(end[:, cs].min() - t0) / 1e3:.1f}..{(end[:, cs].max() - t0) / 1e3:.1f}")
# persistence: per-(rank, CTA) busy time correlation between calls, and per-SM busy
if len(busy_runs) > 1:
    b0, b1 = busy_runs[0].ravel(), busy_runs[1].ravel()
    print(f"busy-time correlation between calls: {np.corrcoef(b0, b1)[0, 1]:.2f}")
smb = {}
for r in range(P):
    for c in range(busy_runs[-1].shape[1]):
        smb.setdefault(int(sm[r, c]), []).append(busy_runs[-1][r, c])
vals = sorted((np.mean(v), s) for s, v in smb.items())
print("slowest SMs (mean busy us):", [(s, round(m / 1e3, 1)) for m, s in vals[-8:]])
print("fastest SMs (mean busy us):", [(s, round(m / 1e3, 1)) for m, s in vals[:8]])
lb.finalize()
# chain analysis: a slice chain = the same CTA index on every rank; its phase pace is set by
# its slowest member.  Compare with chains formed from SMs of neighbouring ids.
b = busy_runs[-1]
chain_max = b.max(axis=0)
print(f"chains by CTA index: max-member busy min {chain_max.min() / 1e3:.1f} med {np.median(chain_max) / 1e3:.1f} "
      f"max {chain_max.max() / 1e3:.1f} us; mean member busy {b.mean() / 1e3:.1f} us")
sm_mean = {s: np.mean(v) for s, v in smb.items()}
ids = sorted(sm_mean)
grp = [ids[i:i + 4] for i in range(0, len(ids), 4)]
gm = np.array([max(sm_mean[s] for s in g) for g in grp])
print(f"hypothetical chains of 4 neighbouring SMs: slowest-SM busy min {gm.min() / 1e3:.1f} med {np.median(gm) / 1e3:.1f} "
      f"max {gm.max() / 1e3:.1f} us; harmonic balance -> {len(gm) / np.sum(1.0 / gm) / 1e3:.1f} us")
print("per-SM mean busy (us) by SM id:", [round(sm_mean[s] / 1e3) for s in ids])
