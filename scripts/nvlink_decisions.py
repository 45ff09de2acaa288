"""Every multi-GPU policy choice that round 1 could only tune on loopback, answered by ONE
multi-GPU lease (VERDICT r01 "next round" 6).

  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
      scripts/nvlink_decisions.py --out-dir gpurun_out/decisions [--only NAME,...]
  (scripts/nvlink_decisions.sh wraps it; DDL_BENCH_SAME_GPU=1 dry-runs it with every rank
  on cuda:0 -- gloo bootstrap, numbers meaningless.)

One CSV per decision, rows `decision,label,P,dims,bytes,us,busbw_GBs,pct_900`:

* crossover   -- LL vs pull one-shot vs hierarchical (forced) from 1 KiB to 8 MiB, dims [P]
                 and the default factorisation: where AUTO's thresholds (64 KiB LL, 512 KiB
                 one-shot; ddl_host.cu) belong on NVLink.
* barriers    -- per-phase barriers (default) vs the streaming variant (DDL_STREAM=1, PATH 5:
                 no inner barriers, per-chunk progress flags), 1-256 MiB.
* tma         -- TMA bulk copies sourcing peer memory (default) vs register-staged loads
                 (DDL_NO_TMA=1), 1-256 MiB: does cp.async.bulk from a cudaIpc-mapped peer work
                 and pay over NVLink?  (Every row is value-checked, so a failing bulk copy
                 shows as a failed gate, not a number.)
* channels    -- the bench step (5 ResNet-50 buckets, grouped) with DDL_CHANNELS 1-4 and L2
                 hints on (15) / off (0).
* waves       -- hierarchical calls in 1 / 2 / 4 / 8 waves (DDL_WAVES) at 32-256 MiB.
* nvls        -- the NVLS phases (multimem, DDL_NVLS_BYTES) on every live dim and on each
                 dim alone (DDL_NVLS_DIMS), 1-256 MiB; a row UNAVAILABLE (with the setup
                 status) where the box cannot create multicast objects.
* barrier_rtt -- the .sys barrier round trip over NVSwitch: tiny hierarchical calls (one
                 16-B vector per block) on dims with 1, 2, 3 live dims (3, 5, 7 barriers);
                 the slope is the cost of one barrier.

Every timed configuration is preceded by a value gate (x_r = r + 1, sum = P(P+1)/2 on every
element; no oracle on this path).  Timing: CUDA-graph replay of `iters` calls, CUDA events,
max over ranks.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_1811_12174_b200 import ddl  # noqa: E402

KIB, MIB = 1 << 10, 1 << 20


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
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


class Ctx:
    def __init__(self, args):
        self.rank, self.world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
        self.same_gpu = os.environ.get("DDL_BENCH_SAME_GPU") == "1"
        dev = 0 if self.same_gpu else int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(dev)
        if self.same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        self.args = args
        self.dev = dev
        self.tdev = "cpu" if self.same_gpu else "cuda"

    def max_over_ranks(self, x):
        t = torch.tensor([x], device=self.tdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def comm(self, dims, env, max_bytes):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            return ddl.init(dims, max_bytes=max_bytes)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


def gated_time(ctx, comm, nbytes, op="sum", iters=None):
    """x_r = r + 1 in the symmetric buffer, value gate, then graph-timed calls."""
    P = ctx.world
    n = nbytes // 4
    t = comm.buffer(n, torch.float32)
    t.fill_(float(ctx.rank + 1))
    comm.all_reduce(t, "sum")
    torch.cuda.synchronize()
    ok = bool((t == P * (P + 1) // 2).all()) and comm.async_error() == ddl.SUCCESS
    bad = ctx.max_over_ranks(0.0 if ok else 1.0)
    if bad:
        return None
    iters = ctx.args.iters or iters or max(3, min(200, int(2e9 // max(nbytes, 1))))
    return ctx.max_over_ranks(time_graph(lambda: comm.all_reduce(t, op), iters))


def row(ctx, out, decision, label, dims_spec, nbytes, us):
    if ctx.rank != 0:
        return
    P = ctx.world
    if us is None:
        print(f"{decision},{label},{P},{dims_spec},{nbytes},GATE_FAILED,,", file=out, flush=True)
        return
    bus = nbytes * 2 * (P - 1) / P / us / 1e3
    print(f"{decision},{label},{P},{dims_spec},{nbytes},{us:.2f},{bus:.2f},{bus / 900 * 100:.1f}", file=out, flush=True)


def default_dims(P):
    return bench.DIMS_FOR_N.get(P, str(P))


def d_crossover(ctx, out):
    P = ctx.world
    sizes = [KIB << j for j in range(14)]          # 1 KiB .. 8 MiB
    for spec in dict.fromkeys([str(P), default_dims(P)]):
        comm = ctx.comm(ddl.parse_dims(spec), {"DDL_LL_MAX_BYTES": str(8 * MIB)}, 16 * MIB)
        for label, algo in (("ll", ddl.ALGO_LL), ("oneshot", ddl.ALGO_ONESHOT), ("hier", ddl.ALGO_HIER)):
            comm.set_algo(algo, 1 << 40 if algo == ddl.ALGO_ONESHOT else 0)
            if algo == ddl.ALGO_LL:
                comm.set_ll_max(8 * MIB)
            for S in sizes:
                if comm.algo_for(S // 4, "float32") != algo:
                    continue           # does not fit that algorithm's buffers
                row(ctx, out, "crossover", label, spec, S, gated_time(ctx, comm, S))
        comm.set_algo(ddl.ALGO_AUTO, 512 * KIB)
        comm.set_ll_max(64 * KIB)
        for S in sizes:
            row(ctx, out, "crossover", "auto", spec, S, gated_time(ctx, comm, S))
        comm.finalize()


def _ab(ctx, out, decision, variants, sizes, specs=None):
    P = ctx.world
    sizes = [S for S in sizes if S <= ctx.args.max_bytes] or [min(sizes)]
    for spec in specs or dict.fromkeys([default_dims(P), str(P)]):
        for label, env in variants:
            comm = ctx.comm(ddl.parse_dims(spec), env, max(sizes) + MIB)
            comm.set_algo(ddl.ALGO_HIER, 0)
            for S in sizes:
                row(ctx, out, decision, label, spec, S, gated_time(ctx, comm, S))
            comm.finalize()


def d_barriers(ctx, out):
    _ab(ctx, out, "barriers", [("per-phase", {}), ("stream", {"DDL_STREAM": "1"}),
                               ("stream-every4", {"DDL_STREAM": "1", "DDL_STREAM_EVERY": "4"})],
        [MIB << j for j in range(0, 9, 2)])


def d_tma(ctx, out):
    _ab(ctx, out, "tma", [("tma", {"DDL_TMA_MIN_SLICE_BYTES": "0"}), ("default", {}), ("ldg", {"DDL_NO_TMA": "1"})],
        [MIB << j for j in range(0, 9, 2)])


def d_waves(ctx, out):
    _ab(ctx, out, "waves", [(f"w{w}", {"DDL_WAVES": str(w), "DDL_MIN_WAVE_SLICE_BYTES": "0"}) for w in (1, 2, 4, 8)],
        [32 * MIB, 128 * MIB, 256 * MIB])


def d_channels(ctx, out):
    P = ctx.world
    spec = default_dims(P)
    host = bench.resnet50_set(ctx.rank)
    S = sum(h.size for h in host) * 4
    for ch in ("1", "2", "3", "4"):
        for hints in ("47", "15", "0"):
            comm = ctx.comm(ddl.parse_dims(spec), {"DDL_CHANNELS": ch, "DDL_L2_HINTS": hints}, S + 8 * MIB)
            off, views = 0, []
            for h in host:
                v = comm.buffer(h.size, torch.float32, off)
                v.fill_(float(ctx.rank + 1))
                views.append(v)
                off += (h.size * 4 + 255) // 256 * 256
            comm.all_reduce_many(views, "sum")
            torch.cuda.synchronize()
            ok = all(bool((v == P * (P + 1) // 2).all()) for v in views)
            us = None if ctx.max_over_ranks(0.0 if ok else 1.0) else \
                ctx.max_over_ranks(time_graph(lambda: comm.all_reduce_many(views, "avg"), ctx.args.iters or 20))
            row(ctx, out, "channels", f"ch{ch}-hints{hints}", spec, S, us)
            comm.finalize()


def d_barrier_rtt(ctx, out):
    P = ctx.world
    specs = [str(P)]
    if P == 8:
        specs += ["2x4", "2x2x2"]
    elif P == 4:
        specs += ["2x2"]
    for spec in specs:
        comm = ctx.comm(ddl.parse_dims(spec), {}, MIB)
        comm.set_algo(ddl.ALGO_HIER, 0)
        nb = len([g for g in ddl.parse_dims(spec) if g > 1])
        for S in (16 * P, 256 * P, 4096 * P):     # one 16-B vector per block, and a little more
            row(ctx, out, "barrier_rtt", f"{2 * nb + 1}-barriers", spec, S, gated_time(ctx, comm, S, iters=200))
        comm.finalize()


def d_nvls(ctx, out):
    """NVLS phases (DDL_NVLS_BYTES): every live dim in the switch, and each dim alone
    (DDL_NVLS_DIMS), against the direct phases on the same sizes.  fp32 results of switch
    phases are checked against the any-order bound on x_r = r + 1 (exact integers: every
    order gives P(P+1)/2), so the value gate holds here too."""
    P = ctx.world
    sizes = [S for S in (MIB << j for j in range(0, 9, 2)) if S <= ctx.args.max_bytes] or [MIB]
    for spec in dict.fromkeys([default_dims(P), str(P)]):
        dims = ddl.parse_dims(spec)
        live = [d for d, g in enumerate(dims) if g > 1]
        masks = [None] + ([str(1 << d) for d in live] if len(live) > 1 else [])
        for mask in masks:
            env = {"DDL_NVLS_BYTES": str(max(sizes) + MIB)}
            if mask:
                env["DDL_NVLS_DIMS"] = mask
            comm = ctx.comm(dims, env, MIB)
            label = f"nvls-mask{mask or 'all'}"
            if comm.nvls_status != "on":
                if ctx.rank == 0:
                    print(f"nvls,{label},{P},{spec},0,UNAVAILABLE,,{comm.nvls_status[:60]}", file=out, flush=True)
                comm.finalize()
                continue
            comm.set_algo(ddl.ALGO_HIER, 0)
            for S in sizes:
                n = S // 4
                t = comm.nvls_buffer(n, torch.float32)
                t.fill_(float(ctx.rank + 1))
                comm.all_reduce(t, "sum")
                torch.cuda.synchronize()
                ok = bool((t == P * (P + 1) // 2).all())
                us = None if ctx.max_over_ranks(0.0 if ok else 1.0) else \
                    ctx.max_over_ranks(time_graph(lambda: comm.all_reduce(t, "sum"),
                                                  ctx.args.iters or max(3, min(200, int(2e9 // S)))))
                row(ctx, out, "nvls", label, spec, S, us)
            comm.finalize()


DECISIONS = {"crossover": d_crossover, "barriers": d_barriers, "tma": d_tma, "channels": d_channels,
             "waves": d_waves, "barrier_rtt": d_barrier_rtt, "nvls": d_nvls}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out-dir", default="gpurun_out/decisions")
    ap.add_argument("--only", default=",".join(DECISIONS))
    ap.add_argument("--iters", type=int, default=0, help="calls per timing (0 = by size); dry runs use 2")
    ap.add_argument("--max-bytes", type=int, default=256 * MIB, help="largest message of the size sweeps")
    args = ap.parse_args()
    ctx = Ctx(args)
    os.makedirs(args.out_dir, exist_ok=True)
    for name in args.only.split(","):
        path = os.path.join(args.out_dir, f"{name}_P{ctx.world}.csv")
        out = open(path, "w") if ctx.rank == 0 else None
        if ctx.rank == 0:
            print("decision,label,P,dims,bytes,us,busbw_GBs,pct_900", file=out, flush=True)
        DECISIONS[name](ctx, out)
        if out:
            out.close()
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
