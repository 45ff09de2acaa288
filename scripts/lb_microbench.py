"""Loopback micro-benchmark: time one all-reduce (P virtual ranks on one GPU) per size.
python scripts/lb_microbench.py --P 8 --dims 2x4 --sizes 31502336 --dtype float32 --op avg
Prints one CSV row per size: lib,P,dims,dtype,bytes,us,algbw_GBs,busbw_GBs,hbm_alg_GBs."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=8)
ap.add_argument("--dims", default="2x4")
ap.add_argument("--sizes", default="31502336")
ap.add_argument("--dtype", default="float32")
ap.add_argument("--op", default="avg")
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--algo", type=int, default=0)
ap.add_argument("--oneshot-max", type=int, default=256 << 10)
ap.add_argument("--graph", action="store_true", help="capture the timed calls in one CUDA graph (no host launch cost)")
a = ap.parse_args()
tdt = {"float32": torch.float32, "bfloat16": torch.bfloat16, "int32": torch.int32}[a.dtype]
w = torch.tensor([], dtype=tdt).element_size()
dims = ddl.parse_dims(a.dims)
lb = ddl.Loopback(a.P, dims)
lb.set_algo(a.algo, a.oneshot_max)
for S in [int(x) for x in a.sizes.split(",")]:
    n = S // w
    bufs = [torch.ones(n, dtype=tdt, device="cuda") for _ in range(a.P)]
    for _ in range(5):
        lb.all_reduce(bufs, a.op if a.dtype != "int32" else "sum")
    torch.cuda.synchronize()
    op = a.op if a.dtype != "int32" else "sum"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(a.iters):
                    lb.all_reduce(bufs, op)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
    else:
        e0.record()
        for _ in range(a.iters):
            lb.all_reduce(bufs, op)
        e1.record()
    torch.cuda.synchronize()
    assert lb.async_error() == 0
    us = e0.elapsed_time(e1) / a.iters * 1e3
    hb = bench.loopback_hbm_bytes(n, a.P, dims, w)
    print(f"{os.path.basename(ddl.LIB_PATH)},{a.P},{a.dims},{a.dtype},{S},{us:.2f},{S/us/1e3:.1f},"
          f"{S*2*(a.P-1)/a.P/us/1e3:.1f},{hb/us/1e3:.1f},ctas={lb.ctas_for(n, a.dtype)}", flush=True)
    del bufs
