"""Two-level all-reduce (inner dims on libddl, outer 'node' dim over a torch.distributed
transport -- gloo here, standing in for the paper's InfiniBand/Ethernet between nodes,
P:L56-60) in real processes on one GPU: bit-exact vs the oracle with dims = inner + [nodes]."""
import os
import socket

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


def _rank_main(rank, world, port, q, inner, nodes):
    import torch.distributed as dist
    import oracle
    import synthetic_inputs as si
    from gpu_util import to_dev, to_host, same_bits
    from paper_1811_12174_b200.multinode import TwoLevelComm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), DDL_TIMEOUT_MS="30000")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        comm = TwoLevelComm(inner, nodes, max_bytes=8 << 20)
        for dtype, kind, op in (("float32", "normal", "avg"), ("int32", "fullrange", "sum"),
                                ("bfloat16", "normal", "avg")):
            n = 8 * world * 3001
            bufs = si.rank_buffers(dtype, kind, n, world, seed=world)
            t = to_dev(bufs[rank], dtype)
            comm.all_reduce(t, op)
            torch.cuda.synchronize()
            want = oracle.allreduce(bufs, comm.dims, dtype, op)[rank]
            res[dtype] = bool(same_bits(to_host(t), want))
        res["err"] = comm.inner.async_error()
        comm.finalize()
    except Exception as e:
        res["exc"] = repr(e)
    q.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.timeout(400)
@pytest.mark.parametrize("world,inner,nodes", [(4, [2], 2), (8, [2, 2], 2), (8, [4], 2)],
                         ids=["2gpu-x-2nodes", "2x2gpu-x-2nodes", "4gpu-x-2nodes"])
def test_two_level_allreduce(world, inner, nodes):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, inner, nodes)) for r in range(world)]
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
        for dtype in ("float32", "int32", "bfloat16"):
            assert out[r][dtype], (r, dtype)
