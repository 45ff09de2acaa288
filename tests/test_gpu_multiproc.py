"""Two real processes (torch.multiprocessing, gloo bootstrap), both on cuda:0: the complete
multi-process bootstrap -- ddl_init, ddl_export_handle, all_gather_object of the cudaIpc
handles, ddl_connect (cudaIpcOpenMemHandle) -- followed by zero-copy and staged
all-reduces checked against the oracle.  On one GPU the two processes' kernels are
time-sliced by the driver, so this proves the IPC mapping and the protocol, not speed."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q, env, dims):
    import torch.distributed as dist
    import oracle
    import synthetic_inputs as si
    from gpu_util import to_dev, to_host, same_bits
    from paper_1811_12174_b200 import ddl
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), DDL_TIMEOUT_MS="20000")
    os.environ.update(env)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        comm = ddl.init(dims, max_bytes=16 << 20)
        for dtype, op in (("float32", "avg"), ("int32", "sum"), ("bfloat16", "sum")):
            kind = "fullrange" if dtype == "int32" else "normal"
            n = 50_003
            bufs = si.rank_buffers(dtype, kind, n, world)
            want = oracle.allreduce(bufs, dims, dtype, op)[rank]
            zc = comm.buffer(n, to_dev(bufs[0][:1], dtype).dtype)
            zc.copy_(to_dev(bufs[rank], dtype))
            st = to_dev(bufs[rank], dtype)
            comm.all_reduce(zc, op)
            comm.all_reduce(st, op)
            torch.cuda.synchronize()
            res[dtype] = (same_bits(to_host(zc), want), same_bits(to_host(st), want))
        # small messages: the LL one-shot (AUTO up to 64 KiB), pushed through the IPC mapping
        ll_ok = []
        for dtype, op in (("float32", "avg"), ("int32", "sum"), ("bfloat16", "sum")):
            kind = "fullrange" if dtype == "int32" else "normal"
            for n in (1, 3, 1001, 16_384):
                ll_ok.append(comm.algo_for(n, dtype) == ddl.ALGO_LL)
                bufs = si.rank_buffers(dtype, kind, n, world, seed=n)
                want = oracle.allreduce(bufs, dims, dtype, op)[rank]
                st = to_dev(bufs[rank], dtype)
                comm.all_reduce(st, op)
                torch.cuda.synchronize()
                ll_ok.append(bool(same_bits(to_host(st), want)))
        res["ll"] = tuple(ll_ok)
        # staged message larger than the workspace: reduced in pieces (ddl.Comm.all_reduce)
        big = si.rank_buffers("float32", "normal", 6_000_001, world, seed=5)
        want = oracle.allreduce_sampled(big, dims, "float32", "avg", np.arange(0, 6_000_001, 997))
        tb = to_dev(big[rank], "float32")
        comm.all_reduce(tb, "avg")
        torch.cuda.synchronize()
        res["big"] = (same_bits(to_host(tb)[::997], want),)
        # registered (cudaIpc-mapped) user buffer: zero-copy all-reduce on a view
        reg = torch.zeros(300_000, device="cuda")
        comm.register(reg)
        rb = si.rank_buffers("float32", "normal", 250_000, world, seed=9)
        view = reg[1024:1024 + 250_000]
        view.copy_(to_dev(rb[rank], "float32"))
        comm.all_reduce(view, "avg")
        torch.cuda.synchronize()
        res["registered"] = (same_bits(to_host(view), oracle.allreduce(rb, dims, "float32", "avg")[rank]),)
        # grouped all-reduce (one launch for the zero-copy buckets, .sys flags across processes):
        # two buckets in the symmetric buffer, one in the registered buffer, one LL-sized, one staged
        gsz = [400_003, 700_000, 120_000, 999, 80_001]
        gb = [si.rank_buffers("float32", "normal", n, world, seed=40 + i) for i, n in enumerate(gsz)]
        views = [comm.buffer(gsz[0], torch.float32, 0), comm.buffer(gsz[1], torch.float32, 1_600_256),
                 reg[4096:4096 + gsz[2]], comm.buffer(gsz[3], torch.float32, 4_800_000),
                 torch.zeros(gsz[4], device="cuda")]
        for v, b in zip(views, gb):
            v.copy_(to_dev(b[rank], "float32"))
        comm.all_reduce_many(views, "avg")
        torch.cuda.synchronize()
        res["grouped"] = tuple(same_bits(to_host(v), oracle.allreduce(b, dims, "float32", "avg")[rank])
                               for v, b in zip(views, gb))
        # NVLS phases (DDL_NVLS_BYTES at init): on one GPU the multicast setup must fall back on
        # every rank (everything above ran on the direct phases); where it is on (an NVSwitch
        # box with one GPU per process), buffers in the NVLS region are checked: int32 exact,
        # fp32 within the any-order bound of the exact sum (oracle.fold_error_bound)
        res["nvls"] = (comm.nvls_status == "on" or comm.nvls_status.startswith("fallback")
                       or "DDL_NVLS_BYTES" not in env,)
        if comm.nvls_status == "on":
            ok = []
            for dtype, op in (("int32", "sum"), ("float32", "avg"), ("bfloat16", "avg")):
                kind = "fullrange" if dtype == "int32" else "normal"
                n = 1 << 20
                bufs = si.rank_buffers(dtype, kind, n, world, seed=77)
                t = comm.nvls_buffer(n, to_dev(bufs[0][:1], dtype).dtype)
                t.copy_(to_dev(bufs[rank], dtype))
                comm.all_reduce(t, op)
                torch.cuda.synchronize()
                got = to_host(t)
                if dtype == "int32":
                    ok.append(same_bits(got, oracle.naive_sum(bufs, "int32")))
                else:
                    y = oracle.bf16_to_f32(got) if dtype == "bfloat16" else got
                    s64, bound = oracle.fold_error_bound(bufs, dims, dtype, op)
                    ok.append(bool(np.all(np.abs(y.astype(np.float64) - s64) <= bound)))
            res["nvls"] = tuple(ok)
        res["err"] = comm.async_error()
        comm.finalize()
    except Exception as e:  # report, don't hang the parent
        res["exc"] = repr(e)
    q.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.timeout(400)
@pytest.mark.parametrize("world,dims,env", [(2, [2], {}), (2, [2], {"DDL_TMA_MIN_SLICE_BYTES": "0"}),
                                            (4, [2, 2], {"DDL_TMA_MIN_SLICE_BYTES": "0"}),
                                            (8, [4, 2], {}),
                                            (2, [2], {"DDL_NVLS_BYTES": str(8 << 20)}),
                                            (4, [2, 2], {"DDL_NVLS_BYTES": str(8 << 20)})],
                         ids=["2-default", "2-tma", "4-2x2-tma", "8-2x4", "2-nvls", "4-2x2-nvls"])
def test_processes_ipc_one_gpu(world, dims, env):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, env, dims)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            r, res = q.get(timeout=360)
            out[r] = res
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert "exc" not in out[r], out[r]
        assert out[r]["err"] == 0
        for dtype in ("float32", "int32", "bfloat16", "ll", "big", "registered", "grouped", "nvls"):
            assert all(out[r][dtype]), (r, dtype)
