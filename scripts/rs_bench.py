"""Reduce-scatter-phase efficiency in loopback: ddl_group_reduce_scatter (RS phases only) at
P = 8, dims 8 / 2x4, fp32, CUDA-graph timed.  HBM bytes per call (schedule): RS phase d reads
g_d * |A_{d+1}| blocks and writes |A_{d+1}| per rank (partials of non-last phases may hit L2);
the compulsory part is every rank's input read once (P * P * recv) plus each rank's result
written once (P * recv)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl
import bench


def time_graph(fn, iters):
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
    return e0.elapsed_time(e1) * 1e3 / iters


peak, src = bench.peaks()
print(f"# HBM peak {peak} ({src})")
print("dims,recv_bytes,us,compulsory_GBs,frac")
for spec in ("8", "2x4"):
    lb = ddl.Loopback(8, ddl.parse_dims(spec))
    for recv in (1 << 20, 1 << 22, 1 << 24):
        sends = [torch.full((8 * recv,), float(r + 1), device="cuda") for r in range(8)]
        outs = [torch.empty(recv, device="cuda") for _ in range(8)]
        lb.reduce_scatter(outs, sends)
        torch.cuda.synchronize()
        assert all(bool((o == 36).all()) for o in outs)
        us = time_graph(lambda: lb.reduce_scatter(outs, sends), 20)
        comp = (8 * 8 * recv + 8 * recv) * 4
        print(f"{spec},{recv * 4},{us:.1f},{comp / us / 1e3:.0f},{comp / us / 1e3 / peak:.3f}", flush=True)
    lb.finalize()
