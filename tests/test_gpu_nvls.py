"""NVLS phases (PATH 7) on one GPU.

A real NVSwitch multicast object needs one GPU per member, so on a 1-GPU box the hardware
path (multimem.ld_reduce / multimem.st) cannot run; what CAN run here:
* the PATH 7 kernel with the NVLS phases' data flow emulated by unicast accesses
  (DDL_NVLS_EMULATE=1): RS phases fold the members in DESCENDING coordinate (an order other
  than the direct path's, as the switch's is unspecified), AG phases PUSH each rank's blocks
  into every member (as multimem.st does) -- which exercises the block / slice selection, the
  push barrier an NVLS allgather needs, and the host dispatch, on loopback and on the
  multi-process launch path, every phase in the "switch" and mixed per phase (DDL_NVLS_DIMS);
  int32 bit-exact vs the oracle, fp32 / bf16 within oracle.fold_error_bound (any fold order);
* the graceful fallback of the real setup (tests/test_gpu_multiproc.py "nvls" cases)."""
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


def check(got, bufs, dims, dtype, op, tag):
    if dtype == "int32":
        want = oracle.naive_sum(bufs, "int32")
        assert same_bits(got, want), (tag, first_diff(got, want))
        return
    s, bound = oracle.fold_error_bound(bufs, dims, dtype, op)
    y = (oracle.bf16_to_f32(got) if dtype == "bfloat16" else got).astype(np.float64)
    err = np.abs(y - s)
    assert np.all(err <= bound), (tag, float((err - bound).max()))


CASES = [(8, [4, 2], None), (8, [2, 2, 2], None), (8, [8], None), (4, [2, 2], None), (6, [3, 2], None),
         (8, [4, 2], "1"), (8, [4, 2], "2"), (8, [2, 2, 2], "5"), (8, [4, 1, 2], None)]
IDS = [f"P{P}-{'.'.join(map(str, d))}-mask{m or 'all'}" for P, d, m in CASES]


@pytest.mark.parametrize("P,dims,mask", CASES, ids=IDS)
def test_nvls_emulated_loopback(P, dims, mask):
    env = {"DDL_NVLS_EMULATE": "1"}
    if mask:
        env["DDL_NVLS_DIMS"] = mask
    lb = with_env(env, lambda: ddl.Loopback(P, dims))
    lb.set_algo(ddl.ALGO_HIER, 0)
    for dtype in ("int32", "float32", "bfloat16"):
        for op in (["sum"] if dtype == "int32" else ["sum", "avg"]):
            for n in (8, 1000, 40_000, 1_000_000):
                bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=n + P)
                dev = [to_dev(b, dtype) for b in bufs]
                lb.all_reduce(dev, op)
                torch.cuda.synchronize()
                assert lb.async_error() == ddl.SUCCESS
                outs = [to_host(t) for t in dev]
                for r in range(P):
                    assert same_bits(outs[r], outs[0]), (dims, dtype, op, n, r)   # replicas identical
                check(outs[0], bufs, dims, dtype, op, (dims, mask, dtype, op, n))
    lb.finalize()


@pytest.mark.parametrize("P,dims,mask", [(8, [4, 2], None), (4, [2, 2], "1"), (8, [2, 2, 2], None), (2, [2], None)])
def test_nvls_emulated_multiprocess_path(P, dims, mask):
    env = {"DDL_NVLS_EMULATE": "1", "DDL_TIMEOUT_MS": "5000"}
    if mask:
        env["DDL_NVLS_DIMS"] = mask
    g = with_env(env, lambda: ddl.InProcessGroup(P, dims, max_bytes=16 << 20))
    g.set_algo(ddl.ALGO_HIER, 0)
    for dtype in ("int32", "float32", "bfloat16"):
        op = "sum" if dtype == "int32" else "avg"
        for n in (4096, 300_000):
            bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=n)
            zc = [g.buffer(r, n, TORCH[dtype], offset_bytes=4096) for r in range(P)]
            for r in range(P):
                zc[r].copy_(to_dev(bufs[r], dtype))
            st = [to_dev(b, dtype) for b in bufs]
            g.all_reduce(zc, op)
            g.all_reduce(st, op)
            torch.cuda.synchronize()
            assert g.async_error() == ddl.SUCCESS
            for name, ts in (("zero-copy", zc), ("staged", st)):
                outs = [to_host(t) for t in ts]
                for r in range(P):
                    assert same_bits(outs[r], outs[0]), (name, dims, dtype, n, r)
                check(outs[0], bufs, dims, dtype, op, (name, dims, dtype, n))
    g.finalize()


def test_nvls_emulated_two_member_phases_bit_exact():
    """With only 2-member groups every fold order is the same (a + b, rounded once), so the
    emulated NVLS path must equal the oracle's direct result bit for bit."""
    lb = with_env({"DDL_NVLS_EMULATE": "1"}, lambda: ddl.Loopback(8, [2, 2, 2]))
    lb.set_algo(ddl.ALGO_HIER, 0)
    for dtype in ("float32", "bfloat16"):
        bufs = si.rank_buffers(dtype, "normal", 123_456, 8, seed=3)
        want = oracle.allreduce(bufs, [2, 2, 2], dtype, "avg")
        dev = [to_dev(b, dtype) for b in bufs]
        lb.all_reduce(dev, "avg")
        torch.cuda.synchronize()
        for r in range(8):
            assert same_bits(to_host(dev[r]), want[r]), (dtype, r)
    lb.finalize()


def test_nvls_emulated_randomized():
    """Random P, factorisation, per-dim NVLS mask, dtype, op and length (16-B multiples and
    ragged, which keep the direct path): int32 exact, fp32 / bf16 within the any-order bound,
    replicas identical."""
    rng = np.random.Generator(np.random.PCG64(77))
    cases = [(2, [2]), (4, [2, 2]), (6, [3, 2]), (8, [4, 2]), (8, [2, 2, 2]), (8, [8]), (16, [4, 4]), (12, [2, 3, 2])]
    for inst in range(20):
        P, dims = cases[int(rng.integers(len(cases)))]
        mask = str(int(rng.integers(1, 1 << len(dims))))
        lb = with_env({"DDL_NVLS_EMULATE": "1", "DDL_NVLS_DIMS": mask}, lambda: ddl.Loopback(P, dims))
        lb.set_algo(ddl.ALGO_HIER, 0)
        dtype = ["int32", "float32", "bfloat16"][int(rng.integers(3))]
        op = "sum" if dtype == "int32" else ["sum", "avg"][int(rng.integers(2))]
        n = int(rng.choice([8, 64, 1000, 4096, 100_000, 100_003, 777_777]))
        bufs = si.rank_buffers(dtype, KIND[dtype], n, P, seed=inst)
        dev = [to_dev(b, dtype) for b in bufs]
        lb.all_reduce(dev, op)
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS
        outs = [to_host(t) for t in dev]
        for r in range(P):
            assert same_bits(outs[r], outs[0]), (inst, dims, mask, dtype, n, r)
        check(outs[0], bufs, dims, dtype, op, (inst, dims, mask, dtype, op, n))
        lb.finalize()


@pytest.mark.parametrize("P,dims", [(8, [4, 2]), (4, [2, 2]), (8, [2, 2, 2])])
def test_nvls_emulated_reduce_scatter_allgather(P, dims):
    """The reduce-scatter and allgather entry points through PATH 7 with the NVLS data flow
    emulated (loopback and the multi-process path): reduce-scatter slices within the
    any-order bound (int32 exact), allgather bit-exact (a pure copy)."""
    recv = 4096 + 64
    lb = with_env({"DDL_NVLS_EMULATE": "1"}, lambda: ddl.Loopback(P, dims))
    g = with_env({"DDL_NVLS_EMULATE": "1", "DDL_TIMEOUT_MS": "5000"},
                 lambda: ddl.InProcessGroup(P, dims, max_bytes=8 << 20))
    for comm in (lb, g):
        for dtype in ("int32", "float32", "bfloat16"):
            op = "sum" if dtype == "int32" else "avg"
            bufs = si.rank_buffers(dtype, KIND[dtype], P * recv, P, seed=11)
            sends = [to_dev(b, dtype) for b in bufs]
            outs = [torch.empty(recv, dtype=TORCH[dtype], device="cuda") for _ in range(P)]
            comm.reduce_scatter(outs, sends, op)
            torch.cuda.synchronize()
            for r in range(P):
                sl = [b[r * recv:(r + 1) * recv] for b in bufs]
                check(to_host(outs[r]), sl, dims, dtype, op, ("rs", type(comm).__name__, dims, dtype, r))
            blocks = si.rank_buffers(dtype, KIND[dtype], recv, P, seed=12)
            want = oracle.allgather(blocks, dims, dtype)
            ins = [to_dev(b, dtype) for b in blocks]
            gat = [torch.empty(P * recv, dtype=TORCH[dtype], device="cuda") for _ in range(P)]
            comm.all_gather(gat, ins)
            torch.cuda.synchronize()
            for r in range(P):
                assert same_bits(to_host(gat[r]), want[r]), ("ag", type(comm).__name__, dims, dtype, r)
    lb.finalize()
    g.finalize()
