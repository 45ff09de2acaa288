"""Run the bench.py N=1 workload (ResNet-50 gradient set, 8 virtual ranks, dims 2x4, avg)
for W warm-up steps + 1 step, nothing else -- the target of the ncu captures (one grouped
launch per step):
  ncu --set full -k regex:ddl_chain -s W -c 1 python scripts/profile_step.py --warmup W
(the loopback step runs the column-chain kernel; DDL_LB_CHAIN=0 and -k regex:ddl_multi profile
the slice kernel instead)"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--dims", default="2x4")
a = ap.parse_args()
P, dims = 8, ddl.parse_dims(a.dims)
lb = ddl.Loopback(P, dims)
host = [bench.resnet50_set(r) for r in range(P)]
bufs = [[torch.from_numpy(host[r][b]).cuda() for r in range(P)] for b in range(len(host[0]))]
for _ in range(a.warmup + 1):   # one bench step = one grouped call (bench.py)
    lb.all_reduce_many(bufs, "avg")
torch.cuda.synchronize()
assert lb.async_error() == 0
print("sizes", [h.size for h in host[0]], "algorithmic bytes/step",
      sum(bench.loopback_hbm_bytes(h.size, P, dims, 4) for h in host[0]))
