"""Synchronous DP-SGD through DDP + the DDL comm hook (two real processes on cuda:0, gloo
process group for DDP's own bootstrap, cudaIpc for DDL): after a few steps every replica
holds the same parameters (S:L441 replica consistency) and they match single-process SGD on
the full batch, whose gradient is the mean of the shards' mean gradients (SPEC dp_trainer's
equivalence check), up to fp32 summation order."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

STEPS, BATCH, DIN, DH = 4, 64, 96, 128


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(DIN, DH), torch.nn.Tanh(), torch.nn.Linear(DH, 1))


def _data():
    g = torch.Generator().manual_seed(1)
    x = torch.randn(STEPS, BATCH, DIN, generator=g)
    y = torch.randn(STEPS, BATCH, 1, generator=g)
    return x, y


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP
    from paper_1811_12174_b200 import ddl
    from paper_1811_12174_b200.ddp import ddl_allreduce_hook, rank_shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), DDL_TIMEOUT_MS="20000")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = ddl.init([world], max_bytes=8 << 20)
        model = DDP(_model().cuda(), device_ids=[0], bucket_cap_mb=0.02)  # several buckets
        model.register_comm_hook(comm, ddl_allreduce_hook)
        opt = torch.optim.SGD(model.parameters(), lr=0.1)
        x, y = _data()
        sh = rank_shard(BATCH, rank, world)
        for s in range(STEPS):
            opt.zero_grad()
            loss = torch.nn.functional.mse_loss(model(x[s, sh].cuda()), y[s, sh].cuda())
            loss.backward()
            opt.step()
        torch.cuda.synchronize()
        params = [p.detach().cpu().numpy() for p in model.module.parameters()]  # by value
        nreg = len(comm._ddp_hook["regs"])
        # a rebuilt bucket (same index, new buffer): the old registration is dropped, the new
        # buffer registered and reduced zero-copy -- the registration count does not grow
        class _Bucket:
            def __init__(self, t, i):
                self.t, self.i = t, i

            def buffer(self):
                return self.t

            def index(self):
                return self.i
        nb = torch.full((5000,), float(rank + 1), device="cuda")
        late = False
        try:            # past the agreement window a changed buffer raises (never a hang)
            ddl_allreduce_hook(comm, _Bucket(nb, 0)).wait()
        except RuntimeError:
            late = True
        comm._ddp_hook["calls"].clear()        # a rebuild inside the agreement window
        ddl_allreduce_hook(comm, _Bucket(nb, 0)).wait()
        torch.cuda.synchronize()
        rebuilt_ok = late and bool((nb == (world + 1) / 2).all()) and len(comm._ddp_hook["regs"]) == nreg
        q.put((rank, params, comm.async_error() if rebuilt_ok else -2))
        comm.finalize()
    except Exception as e:
        q.put((rank, repr(e), -1))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_ddp_hook_matches_full_batch_sgd():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            r, params, err = q.get(timeout=240)
            out[r] = (params, err)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert not isinstance(out[r][0], str), out[r][0]
        assert out[r][1] == 0
    # replicas identical, bit for bit (every rank applies the same averaged gradient)
    for a, b in zip(out[0][0], out[1][0]):
        assert (a == b).all()
    # single-process full-batch SGD reference
    model = _model().cuda()
    opt = torch.optim.SGD(model.parameters(), lr=0.1)
    x, y = _data()
    for s in range(STEPS):
        opt.zero_grad()
        torch.nn.functional.mse_loss(model(x[s].cuda()), y[s].cuda()).backward()
        opt.step()
    for a, b in zip(out[0][0], model.parameters()):
        torch.testing.assert_close(torch.from_numpy(a), b.detach().cpu(), rtol=1e-5, atol=1e-6)
