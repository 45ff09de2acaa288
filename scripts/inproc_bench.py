"""Multi-process launch path on ONE GPU (test hook ddl_debug_connect_local): P communicators
in this process, each rank's all-reduce launched on its own stream (.sys-scope flags, start
and end barriers, per-rank launches), timed like the loopback microbench.  The data stays in
local HBM, so this isolates the protocol/launch overhead of the multi-process path against
loopback mode (one launch, .gpu flags, implied start/end barriers).
python scripts/inproc_bench.py --P 8 --dims 2x4 --sizes 8196000,31502336"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=8)
ap.add_argument("--dims", default="2x4")
ap.add_argument("--sizes", default="8196000,31502336")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--zero-copy", action="store_true")
ap.add_argument("--graph", action="store_true", help="capture all ranks' launches in one CUDA graph")
ap.add_argument("--algo", type=int, default=0)
a = ap.parse_args()
g = ddl.InProcessGroup(a.P, ddl.parse_dims(a.dims), max_bytes=1 << 30)
g.set_algo(a.algo, 512 << 10)
for S in [int(x) for x in a.sizes.split(",")]:
    n = S // 4
    if a.zero_copy:
        bufs = [g.buffer(r, n, torch.float32) for r in range(a.P)]
        for b in bufs:
            b.fill_(1.0)
    else:
        bufs = [torch.ones(n, device="cuda") for _ in range(a.P)]
    for _ in range(3):
        g.all_reduce(bufs, "avg")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.graph:
        cg = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            with torch.cuda.graph(cg, stream=cs):
                for _ in range(a.iters):
                    g.all_reduce(bufs, "avg")
        cg.replay()
        torch.cuda.synchronize()
        e0.record()
        cg.replay()
        e1.record()
    else:
        e0.record()
        for _ in range(a.iters):
            g.all_reduce(bufs, "avg")
        e1.record()
    torch.cuda.synchronize()
    assert g.async_error() == 0
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    print(f"inproc{'-zc' if a.zero_copy else '-staged'}{'-graph' if a.graph else ''}-algo{a.algo},{a.P},{a.dims},{S},{us:.2f},busbw={S*2*(a.P-1)/a.P/us/1e3:.1f}")
g.finalize()
