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


# DDP rebuilds its buckets once, at the start of the second iteration, on every rank at the
# same step.  For the first AGREE_CALLS calls of each bucket the ranks therefore agree
# collectively on whether the bucket's buffer changed (a max over the process group), so
# that all of them -- or none -- enter the collective re-registration even when the rebuilt
# buffer lands at its old address on some ranks only.
AGREE_CALLS = 3


def _any_rank(flag: bool, group) -> bool:
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return bool(t.item())


def ddl_allreduce_hook(state: Comm, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: average the bucket with DDL's all-reduce (enqueued on the current
    stream, so DDP's copy-back is stream-ordered after it).  Each bucket buffer is
    registered with DDL the first time it is seen (a collective every rank performs at the
    same bucket), so every later step all-reduces it zero-copy instead of staging it
    through the workspace.  DDP's buffers are persistent; they change only when DDP rebuilds
    its buckets (after the first iteration), and then the bucket's previous registration is
    dropped before the new buffer is registered -- a stale registration would make a later
    tensor allocated at the old address look zero-copy and read the peers' old buffers.
    Whether to re-register is decided collectively during the first AGREE_CALLS calls of a
    bucket; a buffer that changes later on some rank raises instead of hanging the others."""
    buf = bucket.buffer()
    st = state.__dict__.setdefault("_ddp_hook", {"regs": {}, "calls": {}})
    idx = bucket.index()
    key = (buf.data_ptr(), buf.numel() * buf.element_size())
    have = st["regs"].get(idx)
    changed = have is None or have[0] != key
    ncall = st["calls"].get(idx, 0)
    st["calls"][idx] = ncall + 1
    if ncall < AGREE_CALLS:
        changed = _any_rank(changed, state.group)
    elif changed:
        raise RuntimeError(f"DDL DDP hook: bucket {idx}'s buffer changed after {AGREE_CALLS} calls; "
                           "re-registration is collective and is only agreed on during the first calls")
    if changed:
        if have is not None:
            state.deregister(have[1])
        st["regs"][idx] = (key, state.register(buf))
    state.all_reduce(buf, "avg")
    fut = torch.futures.Future()
    fut.set_result(buf)
    return fut


def rank_shard(n_samples: int, rank: int, world: int) -> slice:
    """The paper's data split: the training set is partitioned across GPUs, not replicated
    (§4.1) -- contiguous equal shards, the remainder dropped."""
    per = n_samples // world
    return slice(rank * per, (rank + 1) * per)
