"""A/B of the loopback kernels at small P (U-Net config 3 at P = 2 and 4, and 64 MiB fp32):
TMA-fed chain (default), LDG chain (DDL_CHAIN_TMA=0), generic chain, slice kernels
(DDL_LB_CHAIN=0); CUDA-graph replay, median of 5, value-checked against the slice kernels."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthetic_inputs as si
from paper_1811_12174_b200 import ddl

VARIANTS = {"tma": {}, "ldg": {"DDL_CHAIN_TMA": "0"}, "generic": {"DDL_CHAIN_GENERIC": "1"}, "slice": {"DDL_LB_CHAIN": "0"}}


def make(P, dims, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return ddl.Loopback(P, dims)
    finally:
        for k, v in old.items():
            os.environ.pop(k, None) if v is None else os.environ.__setitem__(k, v)


def timeit(lb, bufs, reps=20):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                lb.all_reduce(bufs, "avg")
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps * 1e3)
    return statistics.median(ts)


for P, spec, n in [(2, "2", 19_075_523), (2, "2", 16 << 20), (4, "2x2", 19_075_523), (4, "4", 8 << 20), (2, "2", 64 << 20)]:
    dims = ddl.parse_dims(spec)
    host = [torch.from_numpy(si.unet3d_gradients(r, n=n)) for r in range(P)]
    ref = None
    for name, env in VARIANTS.items():
        lb = make(P, dims, env)
        bufs = [h.cuda() for h in host]
        lb.all_reduce(bufs, "avg"); torch.cuda.synchronize()
        if ref is None or name == "slice":
            pass
        out = [b.clone() for b in bufs]
        t = timeit(lb, bufs)
        if name == "tma":
            ref = out
        ok = all(torch.equal(a.view(torch.int32), b.view(torch.int32)) for a, b in zip(out, ref))
        print(f"P={P} {spec:5s} n={n:>10d} {name:8s} {t:8.2f} us  same_as_tma={ok}", flush=True)
        lb.finalize()
