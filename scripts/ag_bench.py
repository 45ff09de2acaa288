"""Allgather-phase efficiency in loopback: ddl_group_allgather (AG phases only, TMA bulk
copy ring) vs a plain device copy of the same output bytes, P = 8, dims 8 / 2x4, CUDA-graph
timed.  Bytes per call: every rank writes P*n elements (its own block through the copy-in,
the P-1 others through the AG phases) and reads them once (sources re-read by P-1 ranks may
hit L2)."""
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


peak, _ = bench.peaks()
print("dims,send_bytes,ag_us,ag_GBs(write+read),copy_us,copy_GBs")
for spec in ("8", "2x4"):
    lb = ddl.Loopback(8, ddl.parse_dims(spec))   # (DDL_* knobs from the environment)
    for n in (1 << 20, 1 << 22, 1 << 24):
        ins = [torch.full((n,), float(r), device="cuda") for r in range(8)]
        outs = [torch.empty(8 * n, device="cuda") for _ in range(8)]
        lb.all_gather(outs, ins)
        torch.cuda.synchronize()
        want = torch.arange(8, device="cuda", dtype=torch.float32).repeat_interleave(n)
        assert all(torch.equal(o, want) for o in outs)
        us = time_graph(lambda: lb.all_gather(outs, ins), 20)
        byts = 2 * 8 * 8 * n * 4
        src = torch.empty(8 * 8 * n, device="cuda")
        dst = torch.empty_like(src)
        cu = time_graph(lambda: dst.copy_(src), 20)
        print(f"{spec},{n * 4},{us:.1f},{byts / us / 1e3:.0f},{cu:.1f},{byts / cu / 1e3:.0f}", flush=True)
    lb.finalize()
