"""Error behaviour of the C ABI on a GPU (include/ddl.h): argument errors return
synchronously and enqueue nothing; the documented codes come back for each misuse."""
import ctypes

import pytest
import torch

from paper_1811_12174_b200 import ddl

pytestmark = pytest.mark.gpu
L = ddl.lib()


def _init(rank, nranks, dims, max_bytes=1 << 20):
    h = ctypes.c_void_p()
    assert L.ddl_init(ctypes.byref(h), rank, nranks, ddl._ints(dims), len(dims), 0, max_bytes) == ddl.SUCCESS
    return h


def test_not_connected_and_finalize():
    h = _init(0, 2, [2])
    t = torch.ones(64, device="cuda")
    assert L.ddl_allreduce(h, t.data_ptr(), 64, ddl.FLOAT32, ddl.SUM, None) == ddl.ERR_NOT_CONNECTED
    assert L.ddl_finalize(h) == ddl.SUCCESS


def test_argument_errors_after_connect():
    hs = [_init(r, 2, [2]) for r in range(2)]
    assert L.ddl_debug_connect_local(ddl._ptrs([h.value for h in hs]), 2) == ddl.SUCCESS
    h = hs[0]
    t = torch.ones(1 << 20, device="cuda")
    ti = torch.ones(64, dtype=torch.int32, device="cuda")
    assert L.ddl_allreduce(h, ti.data_ptr(), 64, ddl.INT32, ddl.AVG, None) == ddl.ERR_UNSUPPORTED
    assert L.ddl_allreduce(h, t.data_ptr() + 4, 64, ddl.FLOAT32, ddl.SUM, None) == ddl.ERR_INVALID_ARGUMENT
    assert L.ddl_allreduce(h, t.data_ptr(), 64, 7, ddl.SUM, None) == ddl.ERR_INVALID_ARGUMENT
    assert L.ddl_allreduce(h, t.data_ptr(), 64, ddl.FLOAT32, 5, None) == ddl.ERR_INVALID_ARGUMENT
    # staged message larger than the 1 MiB workspace
    assert L.ddl_allreduce(h, t.data_ptr(), 1 << 20, ddl.FLOAT32, ddl.SUM, None) == ddl.ERR_TOO_LARGE
    # count 0 is a no-op
    assert L.ddl_allreduce(h, t.data_ptr(), 0, ddl.FLOAT32, ddl.SUM, None) == ddl.SUCCESS
    assert L.ddl_deregister(h, 3) == ddl.ERR_INVALID_ARGUMENT
    torch.cuda.synchronize()
    assert L.ddl_async_error(h) == ddl.SUCCESS
    for x in hs:
        L.ddl_finalize(x)


def test_handle_mismatch():
    """Ranks created with different dims (or sizes) refuse to connect (DDL_ERR_MISMATCH)."""
    a = _init(0, 4, [2, 2])
    b = _init(1, 4, [4])
    hsz = L.ddl_handle_size()
    blobs = []
    for h in (a, b, a, b):
        buf = ctypes.create_string_buffer(hsz)
        assert L.ddl_export_handle(h, buf) == ddl.SUCCESS
        blobs.append(buf.raw)
    # rank fields must match positions: fabricate a 4-rank table from the two exports
    allh = ctypes.create_string_buffer(b"".join(blobs), hsz * 4)
    assert L.ddl_connect(a, allh) in (ddl.ERR_INVALID_ARGUMENT, ddl.ERR_MISMATCH)
    L.ddl_finalize(a)
    L.ddl_finalize(b)


def test_loopback_rejects_multiprocess_calls():
    lb = ddl.Loopback(2, [2])
    t = torch.ones(64, device="cuda")
    assert L.ddl_allreduce(lb.h, t.data_ptr(), 64, ddl.FLOAT32, ddl.SUM, None) == ddl.ERR_INVALID_ARGUMENT
    lb.finalize()


def test_plain_c_program_on_gpu(tmp_path):
    """examples/loopback_allreduce.c: the C ABI driven from C alone (cudaMalloc'd buffers,
    no Python/torch on the data path) reduces correctly on the GPU."""
    import os
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1811_12174_b200")
    exe = tmp_path / "lb"
    subprocess.run(["gcc", "-std=c99", "-O2", "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(root, "examples", "loopback_allreduce.c"), "-L", libdir, "-lddl",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{libdir}:/usr/local/cuda/lib64",
                    "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "loopback_allreduce ok" in r.stdout
