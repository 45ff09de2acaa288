"""Experiment: one all-reduce of S bytes as a single hierarchical call vs the same buffer split
into k contiguous pieces run by the grouped kernel (bit-identical: the result per element
depends only on the fold order of dims).  Loopback, 8 virtual ranks, CUDA-graph replay.
  python scripts/split_single.py --dims 2x4 --sizes 8388608,33554432 --splits 2,4,8"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="2x4")
ap.add_argument("--sizes", default="8388608,33554432,134217728")
ap.add_argument("--splits", default="2,4,8")
a = ap.parse_args()
P, dims = 8, ddl.parse_dims(a.dims)
lb = ddl.Loopback(P, dims)


def timeit(fn, iters=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


for S in [int(x) for x in a.sizes.split(",")]:
    n = S // 4
    bufs = [torch.full((n,), r + 1.0, device="cuda") for r in range(P)]
    row = [f"{S}", f"single {timeit(lambda: lb.all_reduce(bufs, 'sum')):.1f}"]
    for k in [int(x) for x in a.splits.split(",")]:
        step = -(-n // k) // 4 * 4
        pieces = [[b[i:i + step] for b in bufs] for i in range(0, n, step)]
        row.append(f"split{k} {timeit(lambda: lb.all_reduce_many(pieces, 'sum')):.1f}")
    torch.cuda.synchronize()
    print(a.dims, " ".join(row), flush=True)
