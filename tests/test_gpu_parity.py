"""GPU parity: libddl's CUDA path (through the C ABI, loopback mode: P virtual ranks on
one B200, the same kernels and barrier protocol as the multi-process path) against the CPU
oracle, element by element on the same seeded inputs.

Bar (north_star / SURVEY 8(c)): bit-exact for int32, and for fp32 and bf16 under the same
fixed reduction order; all NaNs compare equal.  At full BASELINE sizes the oracle computes
sampled elements (oracle.allreduce_sampled), and properties that hold at any size (all
ranks identical, closed forms) cover the rest.
"""

import numpy as np
import pytest
import torch

import oracle
import synthetic_inputs as si
from gpu_util import to_dev, to_host, same_bits, first_diff
from paper_1811_12174_b200 import ddl

pytestmark = pytest.mark.gpu

KIND = {"int32": "fullrange", "float32": "normal", "bfloat16": "normal"}


def factorisations(P, maxlen=4):
    if P == 1:
        return [[1]]
    out = []

    def rec(rem, cur):
        if rem == 1:
            out.append(list(cur))
            return
        if len(cur) >= maxlen:
            return
        for f in range(2, rem + 1):
            if rem % f == 0:
                rec(rem // f, cur + [f])
    rec(P, [])
    return out


_LB = {}

# loopback kernels: "chain" (default: the column-chain kernel, ddl_chain.cuh) and "slice" (the
# per-CTA slice kernels with device barriers, DDL_LB_CHAIN=0 -- the multi-process path's kernels)
LB_KERNELS = {"chain": {}, "slice": {"DDL_LB_CHAIN": "0"}}


def loopback(P, dims, kernel="chain"):
    import os
    key = (P, tuple(dims), kernel)
    if key not in _LB:
        env = LB_KERNELS[kernel]
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            _LB[key] = ddl.Loopback(P, list(dims))
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    return _LB[key]


def run_allreduce(lb, bufs, dtype, op):
    dev = [to_dev(b, dtype) for b in bufs]
    lb.all_reduce(dev, op)
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS
    return [to_host(t) for t in dev]


def check_allreduce(P, dims, dtype, op, n, algo, seed=1811, kernel="chain"):
    bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=seed)
    want = oracle.allreduce(bufs, dims, dtype, op)
    lb = loopback(P, dims, kernel)
    lb.set_algo(algo, 1 << 40 if algo == ddl.ALGO_ONESHOT else 0)
    got = run_allreduce(lb, bufs, dtype, op)
    for r in range(P):
        assert same_bits(got[r], want[r]), (P, dims, dtype, op, n, algo, kernel, r, first_diff(got[r], want[r]))


CASES = [(P, dims) for P in (2, 3, 4, 6, 8, 16) for dims in factorisations(P)]


@pytest.mark.parametrize("P,dims", CASES, ids=[f"P{P}-{'x'.join(map(str, d))}" for P, d in CASES])
@pytest.mark.parametrize("algo,kernel", [(ddl.ALGO_HIER, "chain"), (ddl.ALGO_HIER, "slice"), (ddl.ALGO_ONESHOT, "chain")],
                         ids=["hier-chain", "hier-slice", "oneshot"])
def test_allreduce_parity(P, dims, algo, kernel):
    sizes = [1, P - 1 if P > 1 else 1, 1000, 40_003]
    for dtype in ("int32", "float32", "bfloat16"):
        for op in (["sum"] if dtype == "int32" else ["sum", "avg"]):
            for n in sizes:
                check_allreduce(P, dims, dtype, op, n, algo, kernel=kernel)


@pytest.mark.parametrize("kernel", sorted(LB_KERNELS))
@pytest.mark.parametrize("P,dims", [(4, [2, 2]), (8, [2, 2, 2]), (8, [8]), (6, [3, 2])])
def test_allreduce_large_ragged(P, dims, kernel):
    for dtype in ("int32", "float32", "bfloat16"):
        check_allreduce(P, dims, dtype, "sum" if dtype == "int32" else "avg", 1_000_003, ddl.ALGO_HIER, kernel=kernel)


def test_auto_algo_switch_is_invisible():
    """mix-and-match (P:L54 (3)): the one-shot and the hierarchy compute the same F_dims,
    so AUTO's choice never changes a bit."""
    P, dims = 8, [4, 2]
    lb = loopback(P, dims)
    for n in (64, 5000, 65_536, 300_000):
        for dtype in ("float32", "bfloat16"):
            bufs = si.rank_buffers(dtype, "normal", n, P, seed=n)
            outs = []
            for algo in (ddl.ALGO_HIER, ddl.ALGO_ONESHOT):
                lb.set_algo(algo, 1 << 40)
                outs.append(run_allreduce(lb, bufs, dtype, "avg"))
            assert all(same_bits(a, b) for a, b in zip(*outs))
    lb.set_algo(ddl.ALGO_AUTO, 512 << 10)


def test_repeated_calls_varying_sizes():
    """Epoch-tagged per-CTA flags: back-to-back calls with different CTA counts and
    algorithms on the same communicator stay correct (no stale flag satisfies a barrier)."""
    P, dims = 8, [2, 2, 2]
    lb = loopback(P, dims)
    lb.set_algo(ddl.ALGO_AUTO, 64 << 10)
    rng = np.random.Generator(np.random.PCG64(5))
    for i in range(40):
        n = int(rng.choice([17, 1000, 4096, 30_000, 200_000, 700_001]))
        bufs = si.rank_buffers("int32", "fullrange", n, P, seed=100 + i)
        got = run_allreduce(lb, bufs, "int32", "sum")
        want = oracle.naive_sum(bufs, "int32")
        assert all(np.array_equal(g, want) for g in got), (i, n)


@pytest.mark.parametrize("P,dims", [(2, [2]), (4, [2, 2]), (4, [4]), (8, [4, 2]), (8, [2, 2, 2]), (6, [2, 3])])
def test_reduce_scatter_allgather(P, dims):
    lb = loopback(P, dims)
    for recv in (96, 1001, 1, 65_536 + 8):
        for dtype in ("int32", "float32", "bfloat16"):
            ops = ["sum"] if dtype == "int32" else ["sum", "avg"]
            for op in ops:
                bufs = si.rank_buffers(dtype, KIND[dtype], P * recv, P, seed=recv)
                want = oracle.reduce_scatter(bufs, dims, dtype, op)
                sends = [to_dev(b, dtype) for b in bufs]
                recvs = [torch.empty(recv, dtype=sends[0].dtype, device="cuda:0") for _ in range(P)]
                lb.reduce_scatter(recvs, sends, op)
                torch.cuda.synchronize()
                for r in range(P):
                    g = to_host(recvs[r])
                    assert same_bits(g, want[r]), (recv, dtype, op, r, first_diff(g, want[r]))
                    assert same_bits(to_host(sends[r]), bufs[r])       # sendbuf untouched
            # allgather of per-rank blocks
            blocks = si.rank_buffers(dtype, KIND[dtype], recv, P, seed=recv + 1)
            want = oracle.allgather(blocks, dims, dtype)
            sends = [to_dev(b, dtype) for b in blocks]
            outs = [torch.full((P * recv,), 7, dtype=sends[0].dtype, device="cuda:0") for _ in range(P)]
            lb.all_gather(outs, sends)
            torch.cuda.synchronize()
            for r in range(P):
                assert same_bits(to_host(outs[r]), want[r]), (recv, dtype, r)


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_local_reduce(dtype):
    for g in (1, 2, 3, 8, 13):
        for n in (1, 1000, (1 << 20) + 5) + (((40 << 20) // 4 + 3,) if g in (3, 8) else ()):
            ins = si.rank_buffers(dtype, KIND[dtype], n, g, seed=g * 7 + n)
            scales = [1.0] if dtype == "int32" else [1.0, 0.125, 1.0 / 3.0]
            for s in scales:
                want = oracle.local_reduce(ins, dtype, s)
                dev = [to_dev(x, dtype) for x in ins]
                out = torch.empty_like(dev[0])
                ddl.local_reduce(dev, out, s)
                torch.cuda.synchronize()
                got = to_host(out)
                assert same_bits(got, want), (g, n, s, first_diff(got, want))


def test_timeout_instead_of_hang():
    """A rank that never arrives makes its peers' barriers time out (sticky
    DDL_ERR_TIMEOUT), never a hang (failure detection)."""
    lb = ddl.Loopback(4, [2, 2])
    lb.set_timeout(200)
    lb.debug_skip_rank(3)
    bufs = [torch.ones(100_000, device="cuda:0") for _ in range(4)]
    lb.all_reduce(bufs)
    torch.cuda.synchronize()
    assert lb.async_error() == ddl.ERR_TIMEOUT
    lb.finalize()


# ------------------------------------------------------------------ BASELINE.json full sizes

def sample_idx(n, k=4096, seed=0):
    rng = np.random.Generator(np.random.PCG64(seed))
    idx = np.unique(np.concatenate([rng.integers(0, n, k), np.arange(min(n, 64)), np.arange(max(0, n - 64), n)]))
    return idx


def check_sampled(bufs, dev, dims, dtype, op):
    idx = sample_idx(len(bufs[0]))
    want = oracle.allreduce_sampled(bufs, dims, dtype, op, idx)
    ti = torch.from_numpy(idx).to("cuda:0")
    for r, t in enumerate(dev):
        got = to_host(t[ti])
        assert same_bits(got, want), (dims, r, first_diff(got, want))
    if dtype == "float32":       # north_star tolerance vs an fp64 naive sum (ledger 8: |y - s| / sum|x|)
        s64, a64 = oracle.exact_sum_f64([np.asarray(b)[idx] for b in bufs], "float32")
        P = len(bufs)
        ref = s64 / P if op == "avg" else s64
        mag = a64 / P if op == "avg" else a64
        y = to_host(dev[0][ti]).astype(np.float64)
        assert np.max(np.abs(y - ref) / np.maximum(mag, 1e-300)) <= 1e-6
    for t in dev[1:]:            # all ranks identical, every element
        assert torch.equal(t.view(torch.int16) if t.dtype == torch.bfloat16 else t,
                           dev[0].view(torch.int16) if t.dtype == torch.bfloat16 else dev[0])


def test_config2_resnet50_buckets_8x_2x4():
    """BASELINE config 2: ResNet-50 gradient set (25.6M fp32 in 5 DDP buckets), avg,
    8 ranks, dims 2x4 = [4, 2]."""
    P, dims = 8, ddl.parse_dims("2x4")
    lb = loopback(P, dims)
    lb.set_algo(ddl.ALGO_AUTO, 512 << 10)
    for b in range(len(si.resnet50_bucket_bytes())):
        bufs = [si.resnet50_bucket(b, r) for r in range(P)]
        dev = [to_dev(x, "float32") for x in bufs]
        lb.all_reduce(dev, "avg")
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS
        check_sampled(bufs, dev, dims, "float32", "avg")


@pytest.mark.parametrize("P,dims", [(2, [2]), (4, [2, 2]), (8, [2, 2, 2])])
def test_config3_unet3d(P, dims):
    lb = loopback(P, dims)
    bufs = [si.unet3d_gradients(r) for r in range(P)]
    dev = [to_dev(x, "float32") for x in bufs]
    lb.all_reduce(dev, "avg")
    torch.cuda.synchronize()
    check_sampled(bufs, dev, dims, "float32", "avg")


@pytest.mark.parametrize("spec", ["8", "2x4", "2x2x2", "4x2"])
def test_config4_bf16_256MiB(spec):
    """BASELINE config 4: bf16 256 MiB, fused x1/8, 8 ranks, dims 8 vs 2x4 vs 2x2x2 (and 4x2)."""
    P, dims = 8, ddl.parse_dims(spec)
    n = (256 << 20) // 2
    bufs = si.rank_buffers("bfloat16", "normal", n, P)
    dev = [to_dev(x, "bfloat16") for x in bufs]
    lb = loopback(P, dims)
    lb.all_reduce(dev, "avg")
    torch.cuda.synchronize()
    check_sampled(bufs, dev, dims, "bfloat16", "avg")
    # secondary tolerance (north_star: bf16 within 1e-2 of an fp64 naive sum, ledger 8)
    idx = sample_idx(n)
    s64, a64 = oracle.exact_sum_f64([b[idx] for b in bufs], "bfloat16")
    y = oracle.bf16_to_f32(to_host(dev[0][torch.from_numpy(idx).cuda()])).astype(np.float64)
    assert np.max(np.abs(y - s64 / P) / np.maximum(a64 / P, 1e-30)) <= 1e-2      # north_star, exactly


def test_int32_bitmask_256MiB_closed_form():
    """int32 bitmask inputs at 256 MiB, 8 ranks, 2x2x2: every element equals the closed
    form (2^P - 1) + P * ((i mod 2^20) << 8) -- a missing/doubled rank or misplaced
    element anywhere shows."""
    P, dims = 8, [2, 2, 2]
    n = (256 << 20) // 4
    dev = [to_dev(si.int32_bitmask(n, r), "int32") for r in range(P)]
    loopback(P, dims).all_reduce(dev)
    torch.cuda.synchronize()
    i = np.arange(n, dtype=np.int64)
    want = ((((1 << P) - 1) + P * ((i % (1 << 20)) << 8)) & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    for t in dev:
        assert np.array_equal(to_host(t), want)


# ------------------------------------------------------------------ alternative kernel paths
PATH_ENVS = {"steal": {"DDL_STEAL": "1"}, "dyn": {"DDL_DYN": "1"}, "ldg": {"DDL_NO_TMA": "1"},
             "tma-all": {"DDL_TMA_MIN_SLICE_BYTES": "0"}, "stream": {"DDL_STREAM": "1"},
             "no-l2-hints": {"DDL_L2_HINTS": "0", "DDL_TMA_MIN_SLICE_BYTES": "0"},
             "no-transpose": {"DDL_TRANSPOSE": "0"},
             "no-deep-copy": {"DDL_DEEP_COPY": "0", "DDL_TMA_MIN_SLICE_BYTES": "0"},
             "no-transpose-waves": {"DDL_TRANSPOSE": "0", "DDL_WAVES": "3", "DDL_MIN_WAVE_SLICE_BYTES": "0"},
             "all-l2-hints": {"DDL_L2_HINTS": "31", "DDL_TMA_MIN_SLICE_BYTES": "0"},
             # waves (TMA-staged path): every CTA walks 3 (5) slices one after another, down to
             # tiny slices
             "waves": {"DDL_WAVES": "3", "DDL_MIN_WAVE_SLICE_BYTES": "0"},
             "waves-tma-all": {"DDL_WAVES": "5", "DDL_MIN_WAVE_SLICE_BYTES": "0", "DDL_TMA_MIN_SLICE_BYTES": "0"}}


EXPERIMENTAL_PATHS = ("steal", "dyn")


@pytest.mark.parametrize("path", sorted(PATH_ENVS))
@pytest.mark.parametrize("P,dims", [(8, [4, 2]), (8, [2, 2, 2]), (8, [8]), (6, [3, 2]), (4, [2, 2])])
def test_kernel_paths_parity(path, P, dims):
    """Every hierarchical kernel variant (register-staged, TMA-staged for all sizes, work
    stealing, rank-level dynamic, streaming, waves) computes the same bits as the oracle."""
    import os
    envs = dict(PATH_ENVS[path], DDL_LB_CHAIN="0")  # variants of the slice kernels
    if path in EXPERIMENTAL_PATHS and not ddl.has_experimental_kernels():
        pytest.skip("PATH 3/4 experiment kernels not compiled (DDL_EXPERIMENTAL=1 bash build.sh)")
    old = {k: os.environ.get(k) for k in envs}
    os.environ.update(envs)
    try:
        lb = ddl.Loopback(P, dims)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    lb.set_algo(ddl.ALGO_HIER, 0)
    for dtype in ("int32", "float32", "bfloat16"):
        for n in (1, 7, 40_003, 1_000_003, 3_000_017):
            op = "sum" if dtype == "int32" else "avg"
            bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=n)
            want = oracle.allreduce(bufs, dims, dtype, op)
            got = run_allreduce(lb, bufs, dtype, op)
            for r in range(P):
                assert same_bits(got[r], want[r]), (path, dims, dtype, n, r, first_diff(got[r], want[r]))
    # reduce-scatter / allgather through the same variant
    recv = 65_536 + 8
    bufs = si.rank_buffers("float32", "normal", P * recv, P, seed=3)
    want = oracle.reduce_scatter(bufs, dims, "float32", "sum")
    sends = [to_dev(b, "float32") for b in bufs]
    outs = [torch.empty(recv, device="cuda") for _ in range(P)]
    lb.reduce_scatter(outs, sends)
    torch.cuda.synchronize()
    assert all(same_bits(to_host(outs[r]), want[r]) for r in range(P))
    lb.finalize()


def test_randomized_instances():
    """SPEC S:L609-style randomized instances on the GPU: random P <= 16, random
    factorisation, dtype, op, algorithm and length (including empty and ragged), bit-exact
    vs the oracle."""
    rng = np.random.Generator(np.random.PCG64(1234))
    for case in range(60):
        P = int(rng.choice([2, 3, 4, 5, 6, 8, 9, 12, 16]))
        fs = factorisations(P)
        dims = fs[int(rng.integers(len(fs)))]
        dtype = ["int32", "float32", "bfloat16"][int(rng.integers(3))]
        op = "sum" if dtype == "int32" else ["sum", "avg"][int(rng.integers(2))]
        n = int(rng.choice([0, 1, 2, 15, 16, 17, 999, 4096, 65_537, 300_001]))
        algo = [ddl.ALGO_AUTO, ddl.ALGO_HIER, ddl.ALGO_ONESHOT][int(rng.integers(3))]
        lb = loopback(P, dims)
        lb.set_algo(algo, 1 << 40 if algo == ddl.ALGO_ONESHOT else 512 << 10)
        bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=case)
        want = oracle.allreduce(bufs, dims, dtype, op) if n else bufs
        got = run_allreduce(lb, bufs, dtype, op)
        for r in range(P):
            assert same_bits(got[r], want[r]), (case, P, dims, dtype, op, n, algo, r)


@pytest.mark.parametrize("algo", [ddl.ALGO_HIER, ddl.ALGO_ONESHOT], ids=["hier", "oneshot"])
def test_cuda_graph_capture_replay(algo):
    """The call epoch lives on the device, so a captured all-reduce can be replayed: every
    replay on fresh inputs matches the oracle (graph-capturable calls)."""
    P, dims, n = 8, [4, 2], 100_003
    lb = ddl.Loopback(P, dims)
    lb.set_algo(algo, 1 << 40)
    bufs = [torch.zeros(n, device="cuda") for _ in range(P)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            lb.all_reduce(bufs, "avg")
            lb.all_reduce(bufs, "sum")   # two calls in one graph
    torch.cuda.synchronize()
    for it in range(4):
        host = si.rank_buffers("float32", "normal", n, P, seed=50 + it)
        for r in range(P):
            bufs[r].copy_(to_dev(host[r], "float32"))
        g.replay()
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS
        mid = oracle.allreduce(host, dims, "float32", "avg")
        want = oracle.allreduce(mid, dims, "float32", "sum")
        for r in range(P):
            assert same_bits(to_host(bufs[r]), want[r]), (it, r)
    lb.finalize()


def test_experiment_kernels_refused_when_not_built():
    """Without DDL_EXPERIMENTAL=1 at build time, asking for PATH 3 / PATH 4 fails loudly at
    init (DDL_ERR_UNSUPPORTED) instead of silently running another kernel."""
    import os
    if ddl.has_experimental_kernels():
        pytest.skip("experiment kernels are compiled in")
    for k in ("DDL_STEAL", "DDL_DYN"):
        os.environ[k] = "1"
        try:
            with pytest.raises(ddl.DDLError) as ei:
                ddl.Loopback(4, [2, 2])
            assert ei.value.code == ddl.ERR_UNSUPPORTED
        finally:
            os.environ.pop(k, None)
