"""Synchronous data-parallel SGD with DDL's all-reduce.

The paper's use of DDL: "DDL can be achieved by adding the 'import ddl' line, using an
MPI-like 'rank' function to specify how data is split across GPUs" (§2.1), gradients
all-reduced every step.  In PyTorch the natural seam is a DistributedDataParallel
communication hook: DDP still buckets the gradients and overlaps communication with the
backward pass; each GradBucket's flat buffer is averaged with ``ddl_allreduce(op=avg)``
(one launch of the hierarchical kernel on the current stream, staged through the
symmetric workspace), instead of NCCL's all-reduce.

    comm = ddl.init("2x4", max_bytes=64 << 20)
    model = DDP(model, device_ids=[local_rank], bucket_cap_mb=25)
    model.register_comm_hook(comm, ddl_allreduce_hook)
"""
import torch
import torch.distributed as dist

from .ddl import Comm


def ddl_allreduce_hook(state: Comm, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: average the bucket with DDL's all-reduce (enqueued on the current
    stream, so DDP's copy-back is stream-ordered after it).  Each bucket buffer is
    registered with DDL the first time it is seen (a collective every rank performs at the
    same bucket), so every later step all-reduces it zero-copy instead of staging it
    through the workspace.  DDP's buffers are persistent; they change only when DDP rebuilds
    its buckets (after the first iteration), and then the bucket's previous registration is
    dropped before the new buffer is registered -- a stale registration would make a later
    tensor allocated at the old address look zero-copy and read the peers' old buffers."""
    buf = bucket.buffer()
    regs = state.__dict__.setdefault("_ddp_registered", {})   # bucket index -> (key, reg_id)
    key = (buf.data_ptr(), buf.numel() * buf.element_size())
    have = regs.get(bucket.index())
    if have is None or have[0] != key:
        if have is not None:
            state.deregister(have[1])
        regs[bucket.index()] = (key, state.register(buf))
    state.all_reduce(buf, "avg")
    fut = torch.futures.Future()
    fut.set_result(buf)
    return fut


def rank_shard(n_samples: int, rank: int, world: int) -> slice:
    """The paper's data split: the training set is partitioned across GPUs, not replicated
    (§4.1) -- contiguous equal shards, the remainder dropped."""
    per = n_samples // world
    return slice(rank * per, (rank + 1) * per)
