"""GPU parity of the LL one-shot (ddl_ll_kernel: flags carried in the
payload) on the multi-process launch path, P communicators in this process on one GPU
(ddl_debug_connect_local): bit-exact vs the oracle for every dtype, op and factorisation,
ragged line tails, multi-CTA messages, epoch/receive-half bookkeeping across calls that
alternate LL with the other algorithms, CUDA-graph replay, and a missing rank -> timeout."""
import os

import numpy as np
import pytest
import torch

import oracle
import synthetic_inputs as si
from gpu_util import to_dev, to_host, same_bits, first_diff, TORCH
from paper_1811_12174_b200 import ddl

pytestmark = pytest.mark.gpu

KIND = {"int32": "fullrange", "float32": "normal", "bfloat16": "normal"}
_G = {}


@pytest.fixture(autouse=True, scope="module")
def _short_timeout():
    old = os.environ.get("DDL_TIMEOUT_MS")
    os.environ["DDL_TIMEOUT_MS"] = "5000"
    yield
    for g in _G.values():
        g.finalize()
    _G.clear()
    if old is None:
        os.environ.pop("DDL_TIMEOUT_MS", None)
    else:
        os.environ["DDL_TIMEOUT_MS"] = old


def group(P, dims):
    key = (P, tuple(dims))
    if key not in _G:
        _G[key] = ddl.InProcessGroup(P, list(dims), max_bytes=16 << 20)
    return _G[key]


CASES = [(2, [2]), (4, [2, 2]), (4, [4]), (8, [4, 2]), (8, [2, 2, 2]), (8, [8]), (6, [3, 2]), (16, [4, 4])]
IDS = [f"P{P}-{'x'.join(map(str, d))}" for P, d in CASES]
# element counts: single element, ragged last lines (bf16: 2/4/6 data bytes; 32-bit: 4),
# one CTA exactly (512 lines), several CTAs, and the 64 KiB default threshold itself
SIZES = {"int32": (1, 3, 1001, 1024, 9_999, 16_384), "float32": (1, 3, 1001, 1024, 9_999, 16_384),
         "bfloat16": (1, 2, 3, 5, 2048, 19_999, 32_768)}


@pytest.mark.parametrize("P,dims", CASES, ids=IDS)
def test_ll_allreduce_parity(P, dims):
    g = group(P, dims)
    g.set_algo(ddl.ALGO_LL, 0)
    for dtype in ("int32", "float32", "bfloat16"):
        for op in (["sum"] if dtype == "int32" else ["sum", "avg"]):
            for n in SIZES[dtype]:
                assert g.algo_for(n, dtype) == ddl.ALGO_LL, (dtype, n)
                bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=n + 3 * P)
                want = oracle.allreduce(bufs, dims, dtype, op)
                zc = [g.buffer(r, n, TORCH[dtype], offset_bytes=256) for r in range(P)]
                for r in range(P):
                    zc[r].copy_(to_dev(bufs[r], dtype))
                st = [to_dev(b, dtype) for b in bufs]
                g.all_reduce(zc, op)
                g.all_reduce(st, op)
                torch.cuda.synchronize()
                assert g.async_error() == ddl.SUCCESS
                for r in range(P):
                    for name, t in (("symmetric", zc[r]), ("plain", st[r])):
                        got = to_host(t)
                        assert same_bits(got, want[r]), (name, dims, dtype, op, n, r, first_diff(got, want[r]))


def test_ll_does_not_touch_past_count():
    """The ragged last line is padded on the wire only: bytes after `count` are untouched."""
    P, dims = 4, [2, 2]
    g = group(P, dims)
    g.set_algo(ddl.ALGO_LL, 0)
    for n in (1, 3, 7):
        big = [torch.full((n + 16,), -7, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
        bufs = si.rank_buffers("bfloat16", "normal", n, P, seed=n)
        for r in range(P):
            big[r][:n].copy_(to_dev(bufs[r], "bfloat16"))
        g.all_reduce([b[:n] for b in big], "sum")
        torch.cuda.synchronize()
        want = oracle.allreduce(bufs, dims, "bfloat16", "sum")
        for r in range(P):
            assert same_bits(to_host(big[r][:n]), want[r])
            assert torch.all(big[r][n:] == -7)


def test_ll_auto_threshold_and_mixed_sequence():
    """AUTO: LL up to the LL threshold, then one-shot, then hierarchical.  A long random
    sequence mixing the three (and both receive halves, both parities of the call counter)
    stays bit-exact: stale words of earlier calls are never taken for this call's data."""
    P, dims = 8, [4, 2]
    g = group(P, dims)
    g.set_algo(ddl.ALGO_AUTO, 512 << 10)
    g.set_ll_max(64 << 10)
    assert g.algo_for(16_384, "float32") == ddl.ALGO_LL
    assert g.algo_for(16_385, "float32") == ddl.ALGO_ONESHOT
    assert g.algo_for(200_000, "float32") == ddl.ALGO_HIER
    rng = np.random.Generator(np.random.PCG64(5))
    for i in range(40):
        n = int(rng.choice([1, 5, 777, 16_384, 16_385, 60_000, 200_000]))
        dtype = ["int32", "float32", "bfloat16"][i % 3]
        op = "sum" if dtype == "int32" else ["sum", "avg"][int(rng.integers(2))]
        bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=100 + i)
        ts = [to_dev(b, dtype) for b in bufs]
        g.all_reduce(ts, op)
        torch.cuda.synchronize()
        want = oracle.allreduce(bufs, dims, dtype, op)
        for r in range(P):
            assert same_bits(to_host(ts[r]), want[r]), (i, n, dtype, op, r)
    assert g.async_error() == ddl.SUCCESS
    g.set_ll_max(0)
    assert g.algo_for(16, "float32") == ddl.ALGO_ONESHOT
    g.set_ll_max(64 << 10)


def test_ll_cuda_graph_replay():
    """LL calls captured in one graph (the call counter lives on the device) replay
    correctly, with the receive half alternating between the captured calls."""
    P, dims, n = 4, [2, 2], 3001
    g = group(P, dims)
    g.set_algo(ddl.ALGO_LL, 0)
    bufs = [torch.zeros(n, device="cuda") for _ in range(P)]
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap):
        with torch.cuda.graph(graph, stream=cap):
            g.all_reduce(bufs, "avg")
            g.all_reduce(bufs, "sum")
            g.all_reduce(bufs, "sum")
    torch.cuda.synchronize()
    for it in range(5):
        host = si.rank_buffers("float32", "normal", n, P, seed=70 + it)
        for r in range(P):
            bufs[r].copy_(to_dev(host[r], "float32"))
        graph.replay()
        torch.cuda.synchronize()
        assert g.async_error() == ddl.SUCCESS
        want = oracle.allreduce(host, dims, "float32", "avg")
        want = oracle.allreduce(want, dims, "float32", "sum")
        want = oracle.allreduce(want, dims, "float32", "sum")
        for r in range(P):
            assert same_bits(to_host(bufs[r]), want[r]), (it, r)


def test_ll_missing_rank_times_out():
    """A rank that never pushes makes its peers' polls time out (sticky DDL_ERR_TIMEOUT)."""
    g = ddl.InProcessGroup(2, [2], max_bytes=1 << 20)
    try:
        g.set_algo(ddl.ALGO_LL, 0)
        L = ddl.lib()
        for h in g.hs:
            assert L.ddl_set_timeout(h, 200) == ddl.SUCCESS
            assert L.ddl_debug_skip_rank(h, 1) == ddl.SUCCESS
        ts = [torch.ones(1000, device="cuda") for _ in range(2)]
        g.all_reduce(ts)
        torch.cuda.synchronize()
        assert g.async_error() == ddl.ERR_TIMEOUT
    finally:
        g.finalize()


@pytest.mark.parametrize("P,dims", CASES + [(8, [4, 1, 2]), (1, [1])],
                         ids=IDS + ["P8-4.1.2", "P1-1"])
def test_ll_loopback_parity(P, dims):
    """The LL kernel in loopback (forced ALGO_LL): all P virtual ranks in one cooperative
    launch, so it also runs under a serialising profiler; bit-exact vs the oracle, and
    repeated calls alternate the receive halves (epoch parity) correctly."""
    lb = ddl.Loopback(P, dims)
    lb.set_algo(ddl.ALGO_LL, 0)
    for dtype in ("int32", "float32", "bfloat16"):
        for op in (["sum"] if dtype == "int32" else ["sum", "avg"]):
            for n in SIZES[dtype]:
                if P > 1:
                    assert lb.algo_for(n, dtype) == ddl.ALGO_LL, (dtype, n)
                bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=n + 5 * P)
                want = oracle.allreduce(bufs, dims, dtype, op)
                dev = [to_dev(b, dtype) for b in bufs]
                lb.all_reduce(dev, op)
                torch.cuda.synchronize()
                assert lb.async_error() == ddl.SUCCESS
                for r in range(P):
                    got = to_host(dev[r])
                    assert same_bits(got, want[r]), (dims, dtype, op, n, r, first_diff(got, want[r]))
    # AUTO in loopback never picks LL (its gain is cross-GPU latency)
    lb.set_algo(ddl.ALGO_AUTO, 512 << 10)
    assert lb.algo_for(1000, "float32") != ddl.ALGO_LL
    lb.finalize()
