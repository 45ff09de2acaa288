"""Loopback small-message latency: LL (forced) vs pull one-shot vs hierarchical, P = 8, dims
8 / 2x4 / 2x2x2, fp32 1 KiB - 256 KiB, CUDA-graph replay of 200 calls (value-gated)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl


def time_graph(fn, iters=200):
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


print("dims,bytes,ll_us,oneshot_us,hier_us")
for spec in ("8", "2x4", "2x2x2"):
    lb = ddl.Loopback(8, ddl.parse_dims(spec))
    for S in [1024 << j for j in range(9)]:
        n = S // 4
        bufs = [torch.full((n,), float(r + 1), device="cuda") for r in range(8)]
        res = []
        for algo in (ddl.ALGO_LL, ddl.ALGO_ONESHOT, ddl.ALGO_HIER):
            lb.set_algo(algo, 1 << 40 if algo == ddl.ALGO_ONESHOT else 0)
            if lb.algo_for(n, "float32") != algo:
                res.append(float("nan"))
                continue
            for b in bufs:
                b.fill_(1.0)
            lb.all_reduce(bufs)
            torch.cuda.synchronize()
            assert all(bool((b == 8).all()) for b in bufs)
            res.append(time_graph(lambda: lb.all_reduce(bufs)))
        print(f"{spec},{S}," + ",".join(f"{x:.2f}" for x in res), flush=True)
    lb.finalize()
