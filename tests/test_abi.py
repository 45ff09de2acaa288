"""CPU tests of the C-ABI boundary (no GPU needed, no compute calls):

* libddl.so loads and exports every function include/ddl.h declares;
* the host planner the kernels share (ddl_plan.h via ddl_plan_* exports) agrees with the
  oracle's independent definitions of groups, block sets, phase traffic and block size;
* argument validation returns the documented error codes without touching a GPU;
* the multi-process bootstrap (handle exchange) works at world_size 2 over gloo.
"""
import os
import re
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1811_12174_b200 import ddl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ddl.h")


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


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ddl_[a-z_]+)\s*\(", text)))


def test_header_symbols_exported():
    names = declared_functions()
    assert len(names) >= 25
    lib = ddl.lib()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding wraps every one of them
    src = open(os.path.join(ROOT, "paper_1811_12174_b200", "ddl.py")).read()
    assert all(f'"{n}"' in src for n in names), [n for n in names if f'"{n}"' not in src]


def test_version_and_strings():
    assert ddl.lib().ddl_version() >= 100
    for code in range(10):
        assert ddl.lib().ddl_result_string(code)
    assert ddl.lib().ddl_result_string(ddl.ERR_TIMEOUT) == b"device barrier timeout"


@pytest.mark.parametrize("P", [1, 2, 3, 4, 6, 8, 12, 16])
def test_planner_matches_oracle(P):
    for dims in factorisations(P):
        assert ddl.check_dims(P, dims) == ddl.SUCCESS
        for r in range(P):
            for d in range(len(dims)):
                assert ddl.plan_group(P, dims, r, d) == oracle.group(r, d, dims)
            for d in range(len(dims) + 1):
                assert ddl.plan_blocks(P, dims, r, d) == oracle.active_blocks(r, d, dims)


@pytest.mark.parametrize("P", [2, 4, 8, 16])
def test_barrier_plan(P):
    """2L+1 barriers; barrier j pairs r with exactly the group that reads r / that r reads
    in the adjacent phases; the end barrier covers every group (every reader of r)."""
    for dims in factorisations(P):
        live = [d for d, g in enumerate(dims) if g > 1]
        L = len(live)
        for r in range(P):
            bars = ddl.plan_barriers(P, dims, r)
            assert len(bars) == 2 * L + 1
            def grp(d):
                return sorted(m for m in oracle.group(r, d, dims) if m != r)
            assert sorted(bars[0]) == grp(live[0])
            for j in range(1, L):
                assert sorted(bars[j]) == grp(live[j])
            assert sorted(bars[L]) == grp(live[-1])
            for jj in range(1, L):
                assert sorted(bars[L + jj]) == grp(live[L - 1 - jj])
            assert sorted(bars[2 * L]) == sorted(m for d in live for m in grp(d))
            # symmetry: if r waits for m in barrier j, m waits for r in barrier j
            for j, peers in enumerate(bars):
                for m in peers:
                    assert r in ddl.plan_barriers(P, dims, m)[j]


@pytest.mark.parametrize("P,n", [(2, 1000), (4, 1_000_003), (8, 8 * 64), (8, 77), (6, 5000), (16, 4096)])
def test_traffic_matches_oracle(P, n):
    for dims in factorisations(P):
        for dtype in ("float32", "bfloat16"):
            t = oracle.Traffic.new(P)
            bufs = [np.zeros(n, dtype=oracle.ddl_oracle.STORAGE[dtype]) for _ in range(P)]
            oracle.allreduce(bufs, dims, dtype, traffic=t)
            for r in range(P):
                rs, ag = ddl.plan_traffic(n, dtype, P, dims, r)
                for d, g in enumerate(dims):
                    assert rs[d] == t.remote_read[r].get(("RS", d), 0), (dims, r, d)
                    assert ag[d] == t.remote_read[r].get(("AG", d), 0), (dims, r, d)


def test_block_elems_matches_oracle():
    for n in [0, 1, 7, 8, 9, 1000, 1_000_003, 25_557_032, 134_217_728]:
        for P in [1, 2, 3, 4, 8, 16]:
            for dt in ("int32", "float32", "bfloat16"):
                assert ddl.block_elems(n, P, dt) == oracle.block_elems(n, P, dt)


def test_bad_dims_codes():
    assert ddl.check_dims(8, [3, 2]) == ddl.ERR_BAD_DIMS
    assert ddl.check_dims(8, [0, 8]) == ddl.ERR_BAD_DIMS
    assert ddl.check_dims(8, [2] * 9) == ddl.ERR_BAD_DIMS
    assert ddl.check_dims(8, [8, 1]) == ddl.SUCCESS                # g_d = 1 allowed


def test_argument_errors_without_gpu():
    import ctypes
    L = ddl.lib()
    h = ctypes.c_void_p()
    assert L.ddl_init(None, 0, 2, ddl._ints([2]), 1, 0, 1 << 20) == ddl.ERR_INVALID_ARGUMENT
    assert L.ddl_init(ctypes.byref(h), 0, 8, ddl._ints([3, 2]), 2, 0, 1 << 20) == ddl.ERR_BAD_DIMS
    assert L.ddl_init(ctypes.byref(h), 0, 32, ddl._ints([32]), 1, 0, 1 << 20) == ddl.ERR_UNSUPPORTED
    assert L.ddl_allreduce(None, None, 10, 0, 0, None) == ddl.ERR_INVALID_ARGUMENT
    assert L.ddl_local_reduce(None, 1, None, 10, 1, 1.0, None) == ddl.ERR_INVALID_ARGUMENT
    assert L.ddl_finalize(None) == ddl.SUCCESS
    assert ddl.parse_dims("2x4") == [4, 2] == oracle.parse_dims("2x4")


# ----------------------------------------------------------------- world_size 2 (gloo)

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # bootstrap exchange with fake handle bytes
        mine = bytes([rank]) * 16
        blob = ddl.exchange_handles([world], mine)
        out["blob"] = blob
        # planner agreement: the owned blocks of all ranks partition the blocks
        owned = ddl.plan_blocks(world, [world], rank, 1)
        allowned = [None] * world
        dist.all_gather_object(allowned, owned)
        out["owned"] = allowned
        # mismatched dims must be rejected on every rank
        try:
            ddl.exchange_handles([world] if rank == 0 else [1, world], mine)
            out["mismatch"] = False
        except ddl.DDLError as e:
            out["mismatch"] = e.code == ddl.ERR_MISMATCH
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bootstrap():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["blob"] == bytes([0]) * 16 + bytes([1]) * 16
        assert sorted(sum(res[r]["owned"], [])) == list(range(world))
        assert res[r]["mismatch"]


def test_plain_c_client(tmp_path):
    """include/ddl.h compiles as C99 and a C program links and runs against libddl.so."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    exe = tmp_path / "c_abi_smoke"
    libdir = os.path.join(ROOT, "paper_1811_12174_b200")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_abi_smoke.c"), "-L", libdir, "-lddl",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "c_abi_smoke ok" in r.stdout


def test_resolve_dims_and_env_override(monkeypatch):
    monkeypatch.delenv("DDL_DIMS", raising=False)
    assert ddl.resolve_dims(None, 8) == [8]
    assert ddl.resolve_dims("2x4", 8) == [4, 2]
    assert ddl.resolve_dims([2, 2, 2], 8) == [2, 2, 2]
    assert ddl.resolve_dims("auto", 8, 4) == [4, 2]
    monkeypatch.setenv("DDL_DIMS", "2x2x2")          # ddlrun-style override
    assert ddl.resolve_dims("2x4", 8) == [2, 2, 2]
    monkeypatch.setenv("DDL_DIMS", "auto")
    assert ddl.resolve_dims(None, 16, 8) == [8, 2]


def test_auto_dims():
    assert ddl.auto_dims(8, 8) == [8]            # one NVSwitch node: flat
    assert ddl.auto_dims(8, 4) == [4, 2]         # "2x4": 2 nodes x 4 GPUs
    assert ddl.auto_dims(16, 8) == [8, 2]
    with pytest.raises(ddl.DDLError):
        ddl.auto_dims(8, 3)


def test_nvls_descriptor_exchange_selftest():
    """The NVLS setup passes POSIX file descriptors between rank processes over abstract Unix
    sockets (SCM_RIGHTS); the library's self-test exchanges a pipe's ends between two
    in-process "ranks" and checks that the received descriptors are the same pipe."""
    assert ddl.lib().ddl_debug_nvls_fd_selftest() == 0
