"""GPU parity of the grouped all-reduce (ddl_allreduce_many / ddl_group_allreduce_many): several
buckets in one launch, split over channels of CTAs.  Every bucket must equal the oracle's
all-reduce of that bucket bit for bit (same fold order as a single call), across
factorisations, dtypes, ragged and one-shot-sized buckets mixed in, more buckets than one
launch holds, every channel count, interleaved with single calls (epoch bookkeeping), on the
loopback and the multi-process launch paths, and under CUDA-graph replay."""
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
# hierarchical-sized buckets (grouped) mixed with one-shot-sized and empty ones (single calls)
SIZES = [300_001, 1_000_003, 7, 2_000_000, 0, 600_000, 123_457]


def with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def check_buckets(devs, hosts, dims, dtype, op, tag):
    P = len(hosts[0])
    for i, (dv, hv) in enumerate(zip(devs, hosts)):
        if hv[0].size == 0:
            continue
        want = oracle.allreduce(hv, dims, dtype, op)
        for r in range(P):
            got = to_host(dv[r])
            assert same_bits(got, want[r]), (tag, i, hv[0].size, r, first_diff(got, want[r]))


def make(P, dtype, sizes, seed):
    hosts = [si.rank_buffers(dtype, KIND[dtype], n, P, seed=seed + i) for i, n in enumerate(sizes)]
    devs = [[to_dev(h, dtype) for h in hv] for hv in hosts]
    return hosts, devs


@pytest.mark.parametrize("kernel", ["chain", "slice"])
@pytest.mark.parametrize("P,dims", [(8, [4, 2]), (8, [2, 2, 2]), (8, [8]), (4, [2, 2]), (6, [3, 2])])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_loopback_grouped_matches_oracle(P, dims, dtype, kernel):
    """The grouped loopback call through the column-chain kernel (default) and through the
    grouped slice kernel (DDL_LB_CHAIN=0, the multi-process path's ddl_multi_kernel)."""
    lb = with_env({"DDL_LB_CHAIN": "0" if kernel == "slice" else "1"}, lambda: ddl.Loopback(P, dims))
    op = "sum" if dtype == "int32" else "avg"
    hosts, devs = make(P, dtype, SIZES, seed=100)
    lb.all_reduce_many(devs, op)
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS
    check_buckets(devs, hosts, dims, dtype, op, "loopback")
    lb.finalize()


@pytest.mark.parametrize("channels,waves,transpose", [("1", "1", "1"), ("3", "1", "1"), ("4", "1", "1"),
                                                       ("2", "3", "1"), ("3", "0", "1"), ("2", "1", "0")])
def test_loopback_grouped_channels_and_split(channels, waves, transpose):
    """11 hierarchical-sized buckets (two launches of <= 8) on 1-4 channels, with and without
    waves per bucket (DDL_GROUP_WAVES, 0 = auto), transposed grid or not."""
    P, dims = 8, [4, 2]
    lb = with_env({"DDL_CHANNELS": channels, "DDL_GROUP_WAVES": waves, "DDL_MIN_WAVE_SLICE_BYTES": "0",
                   "DDL_TRANSPOSE": transpose, "DDL_LB_CHAIN": "0"}, lambda: ddl.Loopback(P, dims))
    sizes = [200_003 + 37_011 * i for i in range(11)]
    hosts, devs = make(P, "float32", sizes, seed=7)
    lb.all_reduce_many(devs, "sum")
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS
    check_buckets(devs, hosts, dims, "float32", "sum", f"channels={channels}")
    lb.finalize()


def test_loopback_grouped_interleaved_with_single_calls():
    """Grouped calls advance the rank epoch by their longest channel's bucket count; single
    calls (hierarchical with waves, one-shot) before and after must still synchronise."""
    P, dims = 8, [4, 2]
    lb = ddl.Loopback(P, dims)
    rng = np.random.Generator(np.random.PCG64(5))
    for it in range(6):
        sizes = [int(x) for x in rng.choice([150_001, 700_000, 1_500_017, 40_000], size=int(rng.integers(2, 6)))]
        hosts, devs = make(P, "int32", sizes, seed=1000 + 10 * it)
        lb.all_reduce_many(devs, "sum")
        n1 = int(rng.choice([1000, 300_000, 9_000_001]))
        single = si.rank_buffers("int32", "fullrange", n1, P, seed=it)
        sd = [to_dev(b, "int32") for b in single]
        lb.all_reduce(sd, "sum")
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS
        check_buckets(devs, hosts, dims, "int32", "sum", f"it={it}")
        want = oracle.naive_sum(single, "int32")
        assert all(np.array_equal(to_host(t), want) for t in sd), it
    lb.finalize()


def test_loopback_grouped_graph_replay():
    P, dims = 8, [2, 2, 2]
    lb = ddl.Loopback(P, dims)
    sizes = [400_000, 1_200_000, 900_001]
    bufs = [[torch.zeros(n, device="cuda") for _ in range(P)] for n in sizes]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            lb.all_reduce_many(bufs, "avg")
    torch.cuda.synchronize()
    for it in range(3):
        hosts = [si.rank_buffers("float32", "normal", n, P, seed=60 + 5 * it + i) for i, n in enumerate(sizes)]
        for b, hv in zip(bufs, hosts):
            for r in range(P):
                b[r].copy_(to_dev(hv[r], "float32"))
        g.replay()
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS
        check_buckets(bufs, hosts, dims, "float32", "avg", f"replay {it}")
    lb.finalize()


@pytest.mark.parametrize("P,dims", [(2, [2]), (4, [2, 2]), (8, [4, 2])])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_multiprocess_path_grouped(P, dims, dtype):
    """The multi-process launch path (P communicators in this process): buckets in the
    symmetric buffer share one launch per rank; a staged bucket and an LL-sized bucket in the
    same call go through single calls."""
    g = with_env({"DDL_TIMEOUT_MS": "5000"}, lambda: ddl.InProcessGroup(P, dims, max_bytes=32 << 20))
    op = "sum" if dtype == "int32" else "avg"
    sizes = [700_001, 1_000, 1_300_000, 300_000, 2_000_003]
    hosts = [si.rank_buffers(dtype, KIND[dtype], n, P, seed=300 + i) for i, n in enumerate(sizes)]
    esz = 4 if dtype != "bfloat16" else 2
    tdt = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}[dtype]
    bufs, off = [], 0
    for i, hv in enumerate(hosts):
        n = hv[0].size
        if i == 3:   # staged (outside the symmetric buffer)
            bufs.append([to_dev(h, dtype) for h in hv])
            continue
        views = [g.buffer(r, n, tdt, off) for r in range(P)]
        for r in range(P):
            views[r].copy_(to_dev(hv[r], dtype))
        bufs.append(views)
        off += (n * esz + 255) // 256 * 256
    g.all_reduce_many(bufs, op)
    torch.cuda.synchronize()
    assert g.async_error() == ddl.SUCCESS
    check_buckets(bufs, hosts, dims, dtype, op, "inproc")
    g.finalize()


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_loopback_grouped_tiny_buckets_forced_hierarchical(dtype):
    """DDL_ALGO=hier sends even 1-element buckets through the grouped kernel: most CTAs get
    empty slices, the rest ragged element-wise tails."""
    P, dims = 8, [2, 2, 2]
    lb = with_env({"DDL_ALGO": "hier"}, lambda: ddl.Loopback(P, dims))
    op = "sum" if dtype == "int32" else "avg"
    hosts, devs = make(P, dtype, [1, 7, 33, 1000, 4097], seed=77)
    lb.all_reduce_many(devs, op)
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS
    check_buckets(devs, hosts, dims, dtype, op, "tiny")
    lb.finalize()


@pytest.mark.parametrize("env", [{"DDL_NO_TMA": "1"}, {"DDL_STREAM": "1"}, {"DDL_STEAL": "1"}],
                         ids=["no-tma", "stream", "steal"])
def test_grouped_honours_kernel_variant(env):
    """DDL_NO_TMA=1 (the register-staged fallback if bulk copies from peer memory fail) and
    the experimental variants hold for all_reduce_many too: every bucket goes through a
    single call of the selected kernel (the grouped kernel is TMA-only), on the
    loopback and the multi-process launch paths, bit-exact vs the oracle."""
    if "DDL_STEAL" in env and not ddl.has_experimental_kernels():
        pytest.skip("PATH 4 not compiled (DDL_EXPERIMENTAL=1 bash build.sh)")
    P, dims = 8, [4, 2]
    lb = with_env(dict(env, DDL_LB_CHAIN="0"), lambda: ddl.Loopback(P, dims))
    hosts, devs = make(P, "float32", SIZES, seed=500)
    lb.all_reduce_many(devs, "avg")
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS
    check_buckets(devs, hosts, dims, "float32", "avg", f"loopback {env}")
    lb.finalize()
    g = with_env(dict(env, DDL_TIMEOUT_MS="5000"), lambda: ddl.InProcessGroup(4, [2, 2], max_bytes=32 << 20))
    sizes = [700_001, 1_300_000, 300_000]
    hosts = [si.rank_buffers("bfloat16", "normal", n, 4, seed=600 + i) for i, n in enumerate(sizes)]
    bufs, off = [], 0
    for hv in hosts:
        n = hv[0].size
        views = [g.buffer(r, n, torch.bfloat16, off) for r in range(4)]
        for r in range(4):
            views[r].copy_(to_dev(hv[r], "bfloat16"))
        bufs.append(views)
        off += (n * 2 + 255) // 256 * 256
    g.all_reduce_many(bufs, "avg")
    torch.cuda.synchronize()
    assert g.async_error() == ddl.SUCCESS
    check_buckets(bufs, hosts, [2, 2], "bfloat16", "avg", f"inproc {env}")
    g.finalize()


def test_reduce_scatter_workspace_growth_refused_in_capture():
    """ddl_group_reduce_scatter grows its workspace on demand; inside a stream
    capture that must be refused (DDL_ERR_TOO_LARGE), not break the capture; after an
    uncaptured call of the size, the captured call works and replays bit-exact."""
    P, dims, recv = 4, [2, 2], 300_000
    lb = ddl.Loopback(P, dims)
    sends = [torch.zeros(P * recv, device="cuda") for _ in range(P)]
    outs = [torch.empty(recv, device="cuda") for _ in range(P)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with pytest.raises(ddl.DDLError) as ei:
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                lb.reduce_scatter(outs, sends)
    assert ei.value.code == ddl.ERR_TOO_LARGE
    torch.cuda.synchronize()
    lb.reduce_scatter(outs, sends)          # grows the workspace outside a capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            lb.reduce_scatter(outs, sends, "avg")
    torch.cuda.synchronize()
    bufs = si.rank_buffers("float32", "normal", P * recv, P, seed=8)
    for r in range(P):
        sends[r].copy_(to_dev(bufs[r], "float32"))
    g.replay()
    torch.cuda.synchronize()
    want = oracle.reduce_scatter(bufs, dims, "float32", "avg")
    for r in range(P):
        assert same_bits(to_host(outs[r]), want[r]), r
    lb.finalize()


def test_grouped_randomized_instances():
    """Randomized grouped all-reduces (SPEC S:L609 style): random P <= 16, factorisation (g_d = 1
    dims included), dtype, op, 1-8 buckets of random (incl. empty / one-shot-sized / ragged)
    lengths, 1-4 channels, 1-3 waves per bucket; every bucket bit-exact vs the oracle."""
    rng = np.random.Generator(np.random.PCG64(4242))
    cases = [(2, [2]), (3, [3]), (4, [2, 2]), (4, [4, 1]), (6, [3, 2]), (8, [4, 2]), (8, [2, 2, 2]), (8, [1, 8]),
             (12, [3, 4]), (16, [4, 4]), (16, [2, 8])]
    for inst in range(24):
        P, dims = cases[int(rng.integers(len(cases)))]
        dtype = ["int32", "float32", "bfloat16"][int(rng.integers(3))]
        op = "sum" if dtype == "int32" else ["sum", "avg"][int(rng.integers(2))]
        nbk = int(rng.integers(1, 9))
        sizes = [int(rng.choice([0, 1, 17, 5000, 70_001, 300_000, 999_983])) for _ in range(nbk)]
        env = {"DDL_CHANNELS": str(int(rng.integers(1, 5))), "DDL_GROUP_WAVES": str(int(rng.integers(1, 4))),
               "DDL_MIN_WAVE_SLICE_BYTES": "0", "DDL_LB_CHAIN": str(inst % 2)}  # slice kernel / chain kernel
        lb = with_env(env, lambda: ddl.Loopback(P, dims))
        hosts, devs = make(P, dtype, sizes, seed=9000 + 10 * inst)
        lb.all_reduce_many(devs, op)
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS, inst
        check_buckets(devs, hosts, dims, dtype, op, f"inst {inst} P={P} dims={dims} {env} sizes={sizes}")
        lb.finalize()
