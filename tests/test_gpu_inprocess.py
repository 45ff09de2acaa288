"""GPU parity of the MULTI-PROCESS kernel path on one B200: P communicators created with
ddl_init (one per rank) in this process, connected with the ddl_debug_connect_local test
hook instead of cudaIpc, each rank's call launched on its own stream so the P kernels run
concurrently.  This exercises what loopback mode does not: per-rank launches, .sys-scope
flags, the symmetric zero-copy buffer at equal offsets, the staged copy-in/copy-out path,
and the staged reduce_scatter / allgather entry points.  Only the cudaIpc mapping itself
(ddl_export_handle / ddl_connect) is not exercised on a 1-GPU box."""
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


def group(P, dims, env=None):
    """env: extra DDL_* settings read at init (e.g. force the TMA-staged path)."""
    key = (P, tuple(dims), tuple(sorted((env or {}).items())))
    if key not in _G:
        old = {k: os.environ.get(k) for k in (env or {})}
        os.environ.update(env or {})
        try:
            _G[key] = ddl.InProcessGroup(P, list(dims), max_bytes=64 << 20)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    return _G[key]


# every hierarchical kernel variant of the multi-process launch path
VARIANTS = {"default": None, "tma": {"DDL_TMA_MIN_SLICE_BYTES": "0"},
            "stream": {"DDL_STREAM": "1", "DDL_TMA_MIN_SLICE_BYTES": "0"},
            "steal": {"DDL_STEAL": "1", "DDL_TMA_MIN_SLICE_BYTES": "0"},
            "check": {"DDL_CHECK": "1"},
            "no-deep-copy": {"DDL_DEEP_COPY": "0", "DDL_TMA_MIN_SLICE_BYTES": "0"},
            "waves": {"DDL_WAVES": "3", "DDL_MIN_WAVE_SLICE_BYTES": "0", "DDL_TMA_MIN_SLICE_BYTES": "0"}}


CASES = [(2, [2]), (4, [2, 2]), (4, [4]), (8, [4, 2]), (8, [2, 2, 2]), (8, [8]), (6, [3, 2])]
IDS = [f"P{P}-{'x'.join(map(str, d))}" for P, d in CASES]


@pytest.mark.parametrize("P,dims", CASES, ids=IDS)
@pytest.mark.parametrize("algo", [ddl.ALGO_HIER, ddl.ALGO_ONESHOT], ids=["hier", "oneshot"])
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_allreduce_zero_copy_and_staged(P, dims, algo, variant):
    if algo == ddl.ALGO_ONESHOT and variant != "default":
        pytest.skip("variants only change the hierarchical kernel")
    if variant == "steal" and not ddl.has_experimental_kernels():
        pytest.skip("PATH 4 not compiled (DDL_EXPERIMENTAL=1 bash build.sh)")
    g = group(P, dims, VARIANTS[variant])
    g.set_algo(algo, 1 << 40 if algo == ddl.ALGO_ONESHOT else 0)
    for dtype in ("int32", "float32", "bfloat16"):
        for op in (["sum"] if dtype == "int32" else ["sum", "avg"]):
            for n in (1, 1000, 40_003, 300_001):
                bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=n + P)
                want = oracle.allreduce(bufs, dims, dtype, op)
                # zero-copy: inside the symmetric buffer, same offset on every rank
                zc = [g.buffer(r, n, TORCH[dtype], offset_bytes=4096) for r in range(P)]
                for r in range(P):
                    zc[r].copy_(to_dev(bufs[r], dtype))
                # staged: ordinary device tensors
                st = [to_dev(b, dtype) for b in bufs]
                g.all_reduce(zc, op)
                g.all_reduce(st, op)
                torch.cuda.synchronize()
                assert g.async_error() == ddl.SUCCESS
                for r in range(P):
                    for name, t in (("zero-copy", zc[r]), ("staged", st[r])):
                        got = to_host(t)
                        assert same_bits(got, want[r]), (name, dims, dtype, op, n, r, first_diff(got, want[r]))


@pytest.mark.parametrize("P,dims", CASES, ids=IDS)
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_reduce_scatter_allgather_staged(P, dims, variant):
    if variant == "steal" and not ddl.has_experimental_kernels():
        pytest.skip("PATH 4 not compiled (DDL_EXPERIMENTAL=1 bash build.sh)")
    g = group(P, dims, VARIANTS[variant])
    for recv in (96, 1001, 50_000):
        for dtype in ("int32", "float32", "bfloat16"):
            op = "sum" if dtype == "int32" else "avg"
            bufs = si.rank_buffers(dtype, KIND[dtype], P * recv, P, seed=recv)
            want = oracle.reduce_scatter(bufs, dims, dtype, op)
            sends = [to_dev(b, dtype) for b in bufs]
            recvs = [torch.empty(recv, dtype=TORCH[dtype], device="cuda") for _ in range(P)]
            g.reduce_scatter(recvs, sends, op)
            torch.cuda.synchronize()
            for r in range(P):
                got = to_host(recvs[r])
                assert same_bits(got, want[r]), (recv, dtype, r, first_diff(got, want[r]))
            blocks = si.rank_buffers(dtype, KIND[dtype], recv, P, seed=recv + 7)
            wantg = oracle.allgather(blocks, dims, dtype)
            sends = [to_dev(b, dtype) for b in blocks]
            outs = [torch.empty(P * recv, dtype=TORCH[dtype], device="cuda") for _ in range(P)]
            g.all_gather(outs, sends)
            torch.cuda.synchronize()
            for r in range(P):
                assert same_bits(to_host(outs[r]), wantg[r]), (recv, dtype, r)
    assert g.async_error() == ddl.SUCCESS


@pytest.mark.parametrize("variant", ["default", "waves"])
def test_many_calls_mixed_paths(variant):
    """Epoch bookkeeping across calls that alternate algorithm, buffer kind and size (waves:
    hierarchical calls advance the rank epoch by their wave count, interleaved with LL and
    one-shot calls whose scratch halves follow the epoch's parity)."""
    P, dims = 4, [2, 2]
    g = group(P, dims, VARIANTS[variant])
    g.set_algo(ddl.ALGO_AUTO, 64 << 10)
    rng = np.random.Generator(np.random.PCG64(11))
    for i in range(30):
        n = int(rng.choice([5, 4000, 16_384, 100_000, 1_000_003]))
        bufs = si.rank_buffers("int32", "fullrange", n, P, seed=i)
        want = oracle.naive_sum(bufs, "int32")
        if i % 2:
            ts = [g.buffer(r, n, torch.int32) for r in range(P)]
            for r in range(P):
                ts[r].copy_(to_dev(bufs[r], "int32"))
        else:
            ts = [to_dev(b, "int32") for b in bufs]
        g.all_reduce(ts)
        torch.cuda.synchronize()
        assert all(np.array_equal(to_host(t), want) for t in ts), (i, n)


@pytest.mark.parametrize("variant", ["default", "tma"])
def test_registered_buffers_zero_copy(variant):
    """ddl_register (in-process hook): all-reduces on registered tensors -- and on views at
    the same offset on every rank -- read peers in place and match the oracle."""
    P, dims = 4, [2, 2]
    g = group(P, dims, VARIANTS[variant])
    n = 2_000_003
    regs = [torch.zeros(n + 64, device="cuda") for _ in range(P)]
    g.register(regs)
    for off, cnt in ((0, n), (64, 500_000), (16, 1)):
        bufs = si.rank_buffers("float32", "normal", cnt, P, seed=off + cnt)
        views = [regs[r][off:off + cnt] for r in range(P)]
        for r in range(P):
            views[r].copy_(to_dev(bufs[r], "float32"))
        g.all_reduce(views, "avg")
        torch.cuda.synchronize()
        want = oracle.allreduce(bufs, dims, "float32", "avg")
        for r in range(P):
            assert same_bits(to_host(views[r]), want[r]), (off, cnt, r)


@pytest.mark.parametrize("variant", ["default", "tma"])
def test_zero_copy_reduce_scatter_allgather(variant):
    """reduce_scatter reading registered send buffers in place, allgather writing registered
    recv buffers in place (symmetric buffer too): bit-exact vs the oracle."""
    P, dims, recv = 8, [4, 2], 70_000
    g = group(P, dims, VARIANTS[variant])
    send = [torch.empty(P * recv, device="cuda") for _ in range(P)]
    g.register(send)
    bufs = si.rank_buffers("float32", "normal", P * recv, P, seed=21)
    for r in range(P):
        send[r].copy_(to_dev(bufs[r], "float32"))
    outs = [torch.empty(recv, device="cuda") for _ in range(P)]
    g.reduce_scatter(outs, send, "avg")
    torch.cuda.synchronize()
    want = oracle.reduce_scatter(bufs, dims, "float32", "avg")
    for r in range(P):
        assert same_bits(to_host(outs[r]), want[r]), ("rs", r)
        assert same_bits(to_host(send[r]), bufs[r])            # send untouched
    # allgather into the symmetric buffer (zero-copy) and into a registered buffer
    blocks = si.rank_buffers("float32", "normal", recv, P, seed=22)
    wantg = oracle.allgather(blocks, dims, "float32")
    sym = [g.buffer(r, P * recv, torch.float32, offset_bytes=1 << 20) for r in range(P)]
    reg = [torch.empty(P * recv, device="cuda") for _ in range(P)]
    g.register(reg)
    for target in (sym, reg):
        ins = [to_dev(b, "float32") for b in blocks]
        g.all_gather(target, ins)
        torch.cuda.synchronize()
        for r in range(P):
            assert same_bits(to_host(target[r]), wantg[r]), ("ag", r)


def test_collective_mismatch_detected():
    """DDL_CHECK=1: ranks calling with different counts get DDL_ERR_MISMATCH (sticky),
    not silent garbage; agreeing calls pass (the 'check' variant above)."""
    os.environ["DDL_TIMEOUT_MS"] = "300"
    try:
        g = group(2, [2], {"DDL_CHECK": "1", "DDL_TIMEOUT_MS": "300"})
    finally:
        os.environ["DDL_TIMEOUT_MS"] = "5000"
    L = ddl.lib()
    ts = [torch.ones(4096, device="cuda") for _ in range(2)]
    counts = [4096, 2048]
    cur = torch.cuda.current_stream()
    for r in range(2):
        g.streams[r].wait_stream(cur)
    for r in range(2):
        assert L.ddl_allreduce(g.hs[r], ts[r].data_ptr(), counts[r], ddl.FLOAT32, ddl.SUM,
                               g.streams[r].cuda_stream) == ddl.SUCCESS
    torch.cuda.synchronize()
    assert g.async_error() == ddl.ERR_MISMATCH
