"""Small loopback / in-process calls for compute-sanitizer (memcheck, racecheck, synccheck):
every kernel variant once on tiny ragged inputs, results checked against the closed form."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl

def check(bufs, want):
    torch.cuda.synchronize()
    assert all(bool((b == want).all()) for b in bufs)

import os
TMA = {"DDL_TMA_MIN_SLICE_BYTES": "0"}     # TMA-staged path even for these tiny slices
WAVES = dict(TMA, DDL_WAVES="3", DDL_MIN_WAVE_SLICE_BYTES="0")   # the wave kernel (PATH 6)
runs = [((4, [2, 2]), {}), ((8, [4, 2]), {}), ((3, [3]), {}),
        ((4, [2, 2]), TMA), ((8, [4, 2]), TMA), ((8, [2, 2, 2]), WAVES)]
for (P, dims), force in runs:
    os.environ.update(force)
    lb = ddl.Loopback(P, dims)
    for k in force:
        os.environ.pop(k, None)
    for algo in (ddl.ALGO_HIER, ddl.ALGO_ONESHOT):
        lb.set_algo(algo, 1 << 30)
        for n in (1, 1003, 70_001):
            for dt in (torch.float32, torch.int32, torch.bfloat16):
                bufs = [torch.full((n,), r + 1, dtype=dt, device="cuda") for r in range(P)]
                lb.all_reduce(bufs)
                check(bufs, P * (P + 1) // 2)
    # reduce-scatter / allgather, aligned and unaligned counts
    for recv in (96, 101):
        sends = [torch.full((P * recv,), r + 1, dtype=torch.float32, device="cuda") for r in range(P)]
        outs = [torch.empty(recv, device="cuda") for _ in range(P)]
        lb.reduce_scatter(outs, sends)
        check(outs, P * (P + 1) // 2)
        ins = [torch.full((recv,), r + 1.0, device="cuda") for r in range(P)]
        g = [torch.empty(P * recv, device="cuda") for _ in range(P)]
        lb.all_gather(g, ins)
        torch.cuda.synchronize()
        want = torch.arange(1, P + 1, device="cuda", dtype=torch.float32).repeat_interleave(recv)
        assert all(torch.equal(x, want) for x in g)
    lb.finalize()
# grouped all-reduce (one launch, channels; waves per bucket too)
for force in ({}, {"DDL_GROUP_WAVES": "2", "DDL_MIN_WAVE_SLICE_BYTES": "0", "DDL_CHANNELS": "3"}):
    os.environ.update(force)
    lb = ddl.Loopback(8, [4, 2])
    for k in force:
        os.environ.pop(k, None)
    bk = [[torch.full((n,), r + 1.0, device="cuda") for r in range(8)] for n in (70_001, 160_003, 99_999, 5)]
    lb.all_reduce_many(bk)
    for b in bk:
        check(b, 36)
    lb.finalize()


def run_group(force):
    """the multi-process launch path (2 in-process communicators): LL, one-shot, hierarchical"""
    os.environ.update(force)
    g = ddl.InProcessGroup(2, [2], max_bytes=1 << 20)
    for k in force:
        os.environ.pop(k, None)
    for algo in (ddl.ALGO_LL, ddl.ALGO_ONESHOT, ddl.ALGO_HIER):
        g.set_algo(algo, 1 << 19)
        for n in (5, 4099):
            for dt in (torch.float32, torch.bfloat16):
                zc = [g.buffer(r, n, dt) for r in range(2)]
                for r in range(2):
                    zc[r].fill_(r + 1)
                st = [torch.full((n,), r + 1.0, dtype=dt, device="cuda") for r in range(2)]
                g.all_reduce(zc)
                g.all_reduce(st)
                check(zc, 3)
                check(st, 3)
    g.finalize()


run_group(TMA)
run_group(WAVES)
# round 2: the LL kernel in loopback (forced), the NVLS kernel (PATH 7) with its data flow
# emulated (every dim in the "switch", and a mixed per-dim mask), g_d = 1 dims
lb = ddl.Loopback(4, [2, 2])
lb.set_algo(ddl.ALGO_LL, 0)
for n in (3, 2049):
    for dt in (torch.float32, torch.bfloat16, torch.int32):
        bufs = [torch.full((n,), r + 1, dtype=dt, device="cuda") for r in range(4)]
        lb.all_reduce(bufs)
        check(bufs, 10)
lb.finalize()
for force in ({"DDL_NVLS_EMULATE": "1"}, {"DDL_NVLS_EMULATE": "1", "DDL_NVLS_DIMS": "2"}):
    os.environ.update(force)
    lb = ddl.Loopback(8, [2, 2, 2])
    for k in force:
        os.environ.pop(k, None)
    lb.set_algo(ddl.ALGO_HIER, 0)
    for n in (8, 70_000):
        for dt in (torch.float32, torch.int32):
            bufs = [torch.full((n,), r + 1, dtype=dt, device="cuda") for r in range(8)]
            lb.all_reduce(bufs)
            check(bufs, 36)
    lb.finalize()
lb = ddl.Loopback(8, [4, 1, 2])
lb.set_algo(ddl.ALGO_HIER, 0)
bufs = [torch.full((1003,), r + 1.0, device="cuda") for r in range(8)]
lb.all_reduce(bufs)
check(bufs, 36)
lb.finalize()
for n in (1001, (32 << 20) // 4 + 3):   # register path, then the TMA-ring path (>= 32 MiB)
    ins = [torch.full((n,), float(j), device="cuda") for j in range(3)]
    out = torch.empty(n, device="cuda")
    ddl.local_reduce(ins, out, 0.5)
    check([out], 1.5)
print("sanitize_check ok")
