"""BASELINE.json configs 3-5 as CSV rows (the single bench.py JSON line covers config 2).

  python scripts/sweep.py --config sweep|bf16|unet3d [--out profiles/x.csv]

* N = 1 (plain python): loopback, P virtual ranks on one B200.
* N > 1 (torchrun): one rank per GPU; NCCL's all_reduce on the same tensor is timed too.

Every row is preceded by a correctness gate: all ranks bit-identical, and for
integer-valued inputs equal to the closed form P*(P+1)/2 (no oracle on this path).
Timing: CUDA-graph replay of `iters` calls (device time, no host launch cost), CUDA events,
max over ranks.  Columns: impl,P,dims,dtype,op,bytes,us,algbw_GBs,busbw_GBs,pct_roof,roof[,sched_pct]
(roof = HBM copy peak for loopback rows -- against the all-reduce's compulsory HBM bytes 2*P*S
(every virtual rank's input read once, its result written once); sched_pct uses the
schedule's phase bytes instead, many of them L2 hits, so it can pass 100 --
and 900 GB/s NVLink for N > 1).  The P = 1 rows of config 5 are the K5 local reduce (g = 8
buffers of S bytes -> 1): algbw column = (g+1)*S / t against the HBM peak.
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_12174_b200 import ddl  # noqa: E402

TD = {"float32": torch.float32, "bfloat16": torch.bfloat16, "int32": torch.int32}


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


def rows_for(config):
    """(P, dims_spec, dtype, op, bytes) per row at loopback P = 8 (or N)."""
    if config == "sweep":         # config 5: fp32 1 KiB .. 1 GiB, sum, at P = 1 / 2 / 4 / 8
        sizes = [1024 << j for j in range(21)]
        rows = [(None, d, "float32", "sum", s) for d in (None, "2x4", "2x2x2") for s in sizes]
        rows += [(P, str(P), "float32", "sum", s) for P in (2, 4) for s in sizes]   # loopback only
        rows += [(1, "k5", "float32", "sum", s) for s in sizes]   # P = 1: the K5 local reduce, g = 8
        return rows
    if config == "bf16":          # config 4: bf16 256 MiB, avg, 8 vs 2x4 vs 2x2x2 (and 4x2)
        return [(8, d, "bfloat16", "avg", 256 << 20) for d in ("8", "2x4", "2x2x2", "4x2")]
    if config == "unet3d":        # config 3: 19,075,523 fp32, avg, 2/4/8 ranks, 2x2x2-style dims
        return [(P, d, "float32", "avg", 19_075_523 * 4) for P, d in ((2, "2"), (4, "2x2"), (8, "2x2x2"))]
    raise SystemExit(f"unknown config {config}")


def k5_row(S, dtype, hbm, out, g=8):
    """P = 1 row of the sweep: out = sum of g local buffers of S bytes (K5), against HBM."""
    w = torch.tensor([], dtype=TD[dtype]).element_size()
    n = S // w
    ins = [torch.full((n,), j + 1, dtype=TD[dtype], device="cuda") for j in range(g)]
    out_t = torch.empty(n, dtype=TD[dtype], device="cuda")
    ddl.local_reduce(ins, out_t)
    torch.cuda.synchronize()
    assert bool((out_t == g * (g + 1) // 2).all()), ("k5", S)
    iters = max(3, min(200, int(2e9 // max(S * (g + 1), 1))))
    us = time_graph(lambda: ddl.local_reduce(ins, out_t), iters)
    hb = (g + 1) * S
    print(",".join(map(str, ["ddl-local-reduce-g8", 1, "-", dtype, "sum", S, f"{us:.2f}", f"{hb / us / 1e3:.2f}", "-",
                             f"{hb / us / 1e3 / hbm * 100:.1f}", "hbm"])), file=out, flush=True)


def loopback(args, out):
    hbm, _ = bench.peaks()
    cache = {}
    for P, spec, dtype, op, S in rows_for(args.config):
        if spec == "k5":
            k5_row(S, dtype, hbm, out)
            continue
        P = P or 8
        spec = spec or str(P)
        dims = ddl.parse_dims(spec)
        w = torch.tensor([], dtype=TD[dtype]).element_size()
        n = S // w
        if P * S > args.max_total_bytes:
            continue
        if (P, spec) not in cache:
            cache[(P, spec)] = ddl.Loopback(P, dims)
        lb = cache[(P, spec)]
        bufs = [torch.full((n,), r + 1, dtype=TD[dtype], device="cuda") for r in range(P)]
        lb.all_reduce(bufs, "sum")
        torch.cuda.synchronize()
        want = P * (P + 1) // 2
        assert all(bool((t == want).all()) for t in bufs), (P, spec, dtype, S)
        iters = max(3, min(200, int(2e9 // max(S * P, 1))))
        us = time_graph(lambda: lb.all_reduce(bufs, op), iters)
        hb = bench.loopback_hbm_bytes(n, P, dims, w)
        algo = "oneshot" if lb.algo_for(n, dtype) == ddl.ALGO_ONESHOT else "hier"
        row = ["ddl-loopback-" + algo, P, spec, dtype, op, S, f"{us:.2f}", f"{S / us / 1e3:.2f}",
               f"{S * 2 * (P - 1) / P / us / 1e3:.2f}", f"{2 * P * S / us / 1e3 / hbm * 100:.1f}", "hbm",
               f"{hb / us / 1e3 / hbm * 100:.1f}"]
        print(",".join(map(str, row)), file=out, flush=True)
        del bufs


def multi(args, out):
    import torch.distributed as dist
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    same_gpu = os.environ.get("DDL_BENCH_SAME_GPU") == "1"   # functional check on one GPU (no NCCL rows)
    torch.cuda.set_device(0 if same_gpu else local)
    if same_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comms = {}
    for P, spec, dtype, op, S in rows_for(args.config):
        if P not in (None, world) or spec == "k5":
            continue
        spec = spec or str(world)
        if math.prod(ddl.parse_dims(spec)) != world:
            continue
        if spec not in comms:
            comms[spec] = ddl.init(spec, max_bytes=args.max_bytes)
        comm = comms[spec]
        w = torch.tensor([], dtype=TD[dtype]).element_size()
        n = S // w
        if S > args.max_bytes:
            continue
        t = comm.buffer(n, TD[dtype])
        t.fill_(rank + 1)
        comm.all_reduce(t, "sum")
        torch.cuda.synchronize()
        assert bool((t == world * (world + 1) // 2).all())
        iters = max(3, min(200, int(2e9 // max(S, 1))))
        dist.barrier()
        us = time_graph(lambda: comm.all_reduce(t, op), iters)
        nus = float("nan")
        if not same_gpu:
            nt = torch.full((n,), rank + 1, dtype=TD[dtype], device="cuda")
            nccl_op = dist.ReduceOp.AVG if op == "avg" else dist.ReduceOp.SUM
            for _ in range(3):
                dist.all_reduce(nt, op=nccl_op)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            e0.record()
            for _ in range(iters):
                dist.all_reduce(nt, op=nccl_op)
            e1.record()
            torch.cuda.synchronize()
            nus = e0.elapsed_time(e1) * 1e3 / iters
        m = torch.tensor([us, nus], device="cpu" if same_gpu else "cuda")
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        us, nus = m.tolist()
        if rank == 0:
            for impl, tt in (("ddl", us), ("nccl", nus)):
                if tt != tt:   # NaN: not measured
                    continue
                bus = S * 2 * (world - 1) / world / tt / 1e3
                print(",".join(map(str, [impl, world, spec, dtype, op, S, f"{tt:.2f}", f"{S / tt / 1e3:.2f}",
                                         f"{bus:.2f}", f"{bus / 900 * 100:.1f}", "nvlink900"])), file=out, flush=True)
    for c in comms.values():
        c.finalize()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sweep", choices=["sweep", "bf16", "unet3d"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--max-total-bytes", type=int, default=24 << 30, help="loopback: cap on P * S")
    ap.add_argument("--max-bytes", type=int, default=(1 << 30) + (1 << 20), help="N > 1: symmetric buffer")
    args = ap.parse_args()
    out = open(args.out, "a") if args.out else sys.stdout
    if int(os.environ.get("RANK", "0")) == 0 and (not args.out or os.path.getsize(args.out) == 0):
        print("impl,P,dims,dtype,op,bytes,us,algbw_GBs,busbw_GBs,pct_roof,roof,sched_pct", file=out, flush=True)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        multi(args, out)
    else:
        loopback(args, out)


if __name__ == "__main__":
    main()
