"""GPU parity of the loopback column-chain kernels (ddl_chain.cuh): the whole
hierarchical schedule (RS phases with the fused epilogue, AG phases) run per column by one
thread -- the compile-time-topology kernels (P = 2, 4, 8) and the generic kernel (any P <= 16,
forced with DDL_CHAIN_GENERIC=1 for the CT topologies too) -- against the CPU oracle and, bit
for bit, against the per-CTA slice kernels with device barriers (DDL_LB_CHAIN=0) on the same
inputs.  Sizes cover the CT kernels' row split: rows whose P columns are all whole vectors
(hot loop), the ragged last block and blocks past n (tail loop), n < P, n < P * vector."""
import os

import numpy as np
import pytest
import torch

import oracle
import synthetic_inputs as si
from gpu_util import to_dev, to_host, same_bits, first_diff
from paper_1811_12174_b200 import ddl

pytestmark = pytest.mark.gpu

KIND = {"int32": "fullrange", "float32": "normal", "bfloat16": "normal"}
KERNELS = {"ct": {"DDL_LB_CHAIN": "1", "DDL_CHAIN_TMA": "0"}, "tma": {"DDL_LB_CHAIN": "1", "DDL_CHAIN_TMA": "1"},
           "generic": {"DDL_LB_CHAIN": "1", "DDL_CHAIN_GENERIC": "1"}, "slice": {"DDL_LB_CHAIN": "0"}}


def make_lb(P, dims, kernel):
    env = KERNELS[kernel]
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        lb = ddl.Loopback(P, dims)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    lb.set_algo(ddl.ALGO_HIER, 0)
    return lb


def run(lb, bufs, dtype, op):
    dev = [to_dev(b, dtype) for b in bufs]
    lb.all_reduce(dev, op)
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS
    return [to_host(t) for t in dev]


def edge_sizes(P, w):
    """Lengths around the row split of a CT kernel: q = roundup(ceil(n/P), V), V = 16/w."""
    V = 16 // w
    out = {1, 2, V - 1, V, V + 1, P - 1, P, P * V - 1, P * V, P * V + 1, 3 * P * V + 5}
    for q in (V, 7 * V, 64 * V):
        for d in (-V - 1, -1, 0, 1):
            out.add(max(1, P * q + d))
            out.add(max(1, (P - 1) * q + d))
    return sorted(out)


TOPOS = [(2, [2]), (4, [4]), (4, [2, 2]), (8, [8]), (8, [4, 2]), (8, [2, 4]), (8, [2, 2, 2]),
         (8, [4, 1, 2]), (6, [3, 2]), (12, [3, 4]), (16, [4, 4]), (16, [2, 2, 2, 2])]


@pytest.mark.parametrize("kernel", ["ct", "tma", "generic"])
@pytest.mark.parametrize("P,dims", TOPOS, ids=[f"P{P}-{'x'.join(map(str, d))}" for P, d in TOPOS])
def test_chain_matches_oracle_edge_sizes(P, dims, kernel):
    lb = make_lb(P, dims, kernel)
    for dtype in ("int32", "float32", "bfloat16"):
        w = 2 if dtype == "bfloat16" else 4
        for op in (["sum"] if dtype == "int32" else ["sum", "avg"]):
            for n in edge_sizes(P, w):
                bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=n + 17)
                want = oracle.allreduce(bufs, dims, dtype, op)
                got = run(lb, bufs, dtype, op)
                for r in range(P):
                    assert same_bits(got[r], want[r]), (kernel, dims, dtype, op, n, r, first_diff(got[r], want[r]))
    lb.finalize()


@pytest.mark.parametrize("P,dims", [(8, [4, 2]), (8, [2, 2, 2]), (8, [8]), (4, [2, 2]), (2, [2]), (6, [3, 2])])
def test_chain_equals_slice_kernels_bitwise(P, dims):
    """Same fold order and rounding points as the barrier kernels: identical bits on several
    million elements per rank (all three kernels, every dtype)."""
    lbs = {k: make_lb(P, dims, k) for k in KERNELS}
    for dtype in ("int32", "float32", "bfloat16"):
        op = "sum" if dtype == "int32" else "avg"
        n = 3_000_017
        bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=99)
        outs = {k: run(lb, bufs, dtype, op) for k, lb in lbs.items()}
        for k in ("ct", "tma", "generic"):
            for r in range(P):
                assert same_bits(outs[k][r], outs["slice"][r]), (k, dims, dtype, r, first_diff(outs[k][r], outs["slice"][r]))
    for lb in lbs.values():
        lb.finalize()


@pytest.mark.parametrize("kernel", ["ct", "tma", "generic"])
def test_chain_grouped_many_buckets(kernel):
    """Grouped calls through the chain kernel: 11 buckets (two launches of <= 8), ragged and
    one-shot-sized ones mixed in, every bucket vs the oracle; and a CUDA-graph replay."""
    P, dims = 8, [4, 2]
    lb = make_lb(P, dims, kernel)
    lb.set_algo(ddl.ALGO_AUTO, 512 << 10)
    sizes = [200_003 + 37_011 * i for i in range(9)] + [7, 40_000]
    hosts = [si.rank_buffers("float32", "normal", n, P, seed=300 + i) for i, n in enumerate(sizes)]
    devs = [[to_dev(h, "float32") for h in hv] for hv in hosts]
    lb.all_reduce_many(devs, "avg")
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS
    for i, hv in enumerate(hosts):
        want = oracle.allreduce(hv, dims, "float32", "avg")
        for r in range(P):
            assert same_bits(to_host(devs[i][r]), want[r]), (kernel, i, r)
    # graph capture + replay on fresh inputs
    bufs = [[torch.zeros(n, device="cuda") for _ in range(P)] for n in sizes[:4]]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            lb.all_reduce_many(bufs, "sum")
    torch.cuda.synchronize()
    for it in range(2):
        hv = [si.rank_buffers("float32", "normal", n, P, seed=500 + 10 * it + i) for i, n in enumerate(sizes[:4])]
        for b, h in zip(bufs, hv):
            for r in range(P):
                b[r].copy_(to_dev(h[r], "float32"))
        g.replay()
        torch.cuda.synchronize()
        for b, h in zip(bufs, hv):
            want = oracle.allreduce(h, dims, "float32", "sum")
            assert all(same_bits(to_host(b[r]), want[r]) for r in range(P)), it
    lb.finalize()


def test_chain_closed_forms_large():
    """Closed forms at 64 Mi elements per rank (every element checked on the device): int32
    rank bitmask sum (a missing or doubled rank shows in the low byte, a misplaced element in
    the high bits), fp32 x_r = r + 1 avg = (P + 1) / 2 exactly."""
    P, dims = 8, [4, 2]
    lb = make_lb(P, dims, "ct")
    n = 64 << 20
    i = torch.arange(n, device="cuda", dtype=torch.int64)
    dev = [((1 << r) | ((i % (1 << 20)) << 8)).to(torch.int32) for r in range(P)]
    lb.all_reduce(dev, "sum")
    want = ((((1 << P) - 1) + P * ((i % (1 << 20)) << 8)) & 0xFFFFFFFF)
    want = torch.where(want >= 1 << 31, want - (1 << 32), want).to(torch.int32)
    torch.cuda.synchronize()
    for t in dev:
        assert torch.equal(t, want)
    del dev, want, i
    f = [torch.full((n,), float(r + 1), device="cuda") for r in range(P)]
    lb.all_reduce(f, "avg")
    torch.cuda.synchronize()
    for t in f:
        assert bool((t == (P + 1) / 2).all())
    lb.finalize()


@pytest.mark.parametrize("kernel", sorted(KERNELS))
@pytest.mark.parametrize("P,dims", [(8, [4, 2]), (8, [2, 2, 2]), (4, [4]), (6, [3, 2]), (16, [4, 4])])
def test_no_write_outside_the_buffers(P, dims, kernel):
    """Own bounds check (compute-sanitizer is disabled on the GPU pool): every rank's buffer is
    a view into a larger allocation whose guard zones before and after hold a canary pattern;
    after all-reduces of ragged lengths (and a grouped call) the guards are bit-identical and
    the results match the oracle -- no kernel writes outside [ptr, ptr + n*w)."""
    lb = make_lb(P, dims, kernel)
    G = 4096 + 8  # guard elements on each side (16-B aligned views: G*w is a multiple of 16)
    for dtype in ("float32", "bfloat16", "int32"):
        w = 2 if dtype == "bfloat16" else 4
        op = "sum" if dtype == "int32" else "avg"
        tdt = {"float32": torch.float32, "bfloat16": torch.bfloat16, "int32": torch.int32}[dtype]
        sizes = [1, 7, 1000, 65_537, 300_001]
        hosts = [si.rank_buffers(dtype, KIND[dtype], n, P, seed=n + 5) for n in sizes]
        bigs, views = [], []
        for n, hv in zip(sizes, hosts):
            bk, vk = [], []
            for r in range(P):
                big = torch.randint(-2**31, 2**31 - 1, ((n + 2 * G) * w // 4 + 1,), dtype=torch.int32,
                                    device="cuda").view(torch.uint8)[: (n + 2 * G) * w].view(tdt)
                v = big[G:G + n]
                v.copy_(to_dev(hv[r], dtype))
                bk.append(big)
                vk.append(v)
            bigs.append(bk)
            views.append(vk)
        guards = [[(b[:G].clone(), b[G + n:].clone()) for b in bk] for n, bk in zip(sizes, bigs)]
        for vk in views[:3]:
            lb.all_reduce(vk, op)
        lb.all_reduce_many(views[3:], op)
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS
        for i, (n, bk) in enumerate(zip(sizes, bigs)):
            want = oracle.allreduce(hosts[i], dims, dtype, op)
            for r in range(P):
                g0, g1 = guards[i][r]
                assert torch.equal(bk[r][:G].view(torch.uint8), g0.view(torch.uint8)), (kernel, dtype, n, r, "before")
                assert torch.equal(bk[r][G + n:].view(torch.uint8), g1.view(torch.uint8)), (kernel, dtype, n, r, "after")
                assert same_bits(to_host(views[i][r]), want[r]), (kernel, dtype, n, r)
    lb.finalize()


def test_first_call_inside_graph_capture(tmp_path):
    """A fresh process whose FIRST loopback all-reduce is captured into a CUDA graph (kernel
    loading, occupancy query and smem attribute happen during the capture): the replay is
    bit-exact vs the oracle, for the TMA-fed chain kernel of 2x4 and the grouped call."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np, torch
import oracle, synthetic_inputs as si
from gpu_util import to_dev, to_host, same_bits
from paper_1811_12174_b200 import ddl
P, dims = 8, [4, 2]
lb = ddl.Loopback(P, dims)
sizes = [300_001, 65_536]
bufs = [[torch.zeros(n, device="cuda") for _ in range(P)] for n in sizes]
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        lb.all_reduce(bufs[0], "avg")
        lb.all_reduce_many(bufs, "sum")
torch.cuda.synchronize()
hv = [si.rank_buffers("float32", "normal", n, P, seed=70 + i) for i, n in enumerate(sizes)]
for b, h in zip(bufs, hv):
    for r in range(P):
        b[r].copy_(to_dev(h[r], "float32"))
g.replay(); torch.cuda.synchronize()
w0 = oracle.allreduce(oracle.allreduce(hv[0], dims, "float32", "avg"), dims, "float32", "sum")
w1 = oracle.allreduce(hv[1], dims, "float32", "sum")
assert lb.async_error() == ddl.SUCCESS
assert all(same_bits(to_host(bufs[0][r]), w0[r]) for r in range(P))
assert all(same_bits(to_host(bufs[1][r]), w1[r]) for r in range(P))
print("capture ok")
''' % (root, os.path.join(root, "tests"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "capture ok" in r.stdout, (r.stdout + r.stderr)[-3000:]


def test_bench_step_every_element_vs_oracle():
    """bench.py N = 1's exact call -- Loopback(8, 2x4).all_reduce_many(the 5 ResNet-50
    buckets, avg), 25.6 M fp32 per virtual rank, through the default (TMA-fed chain) kernel --
    compared with the oracle on EVERY element of every bucket and rank (the oracle runs the
    whole set in ~1 s), plus a second step on the reduced values."""
    P, dims = 8, ddl.parse_dims("2x4")
    lb = ddl.Loopback(P, dims, device=0)
    nb = len(si.resnet50_bucket_bytes())
    host = [[si.resnet50_bucket(b, r) for r in range(P)] for b in range(nb)]
    bufs = [[to_dev(host[b][r], "float32") for r in range(P)] for b in range(nb)]
    for step in range(2):
        lb.all_reduce_many(bufs, "avg")
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS
        for b in range(nb):
            want = oracle.allreduce(host[b], dims, "float32", "avg")
            for r in range(P):
                got = to_host(bufs[b][r])
                assert same_bits(got, want[r]), (step, b, r, first_diff(got, want[r]))
        host = [[w for w in oracle.allreduce(host[b], dims, "float32", "avg")] for b in range(nb)]
    lb.finalize()


@pytest.mark.parametrize("P,spec", [(2, "2"), (4, "2x2"), (8, "2x2x2")])
def test_config3_unet3d_every_element_vs_oracle(P, spec):
    """BASELINE config 3 (3D U-Net gradient set, 19,075,523 fp32, avg) at P = 2 / 4 / 8 through
    the default loopback kernel, every element of every rank vs the oracle."""
    dims = ddl.parse_dims(spec)
    lb = ddl.Loopback(P, dims, device=0)
    host = [si.unet3d_gradients(r) for r in range(P)]
    dev = [to_dev(h, "float32") for h in host]
    lb.all_reduce(dev, "avg")
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS
    want = oracle.allreduce(host, dims, "float32", "avg")
    for r in range(P):
        got = to_host(dev[r])
        assert same_bits(got, want[r]), (spec, r, first_diff(got, want[r]))
    lb.finalize()
