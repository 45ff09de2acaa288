"""Synthetic synchronous DP-SGD step time (the paper's Table 1 use of DDL), with
DDP's gradient buckets all-reduced by DDL (comm hook) or by NCCL (default).

  torchrun --nproc-per-node N scripts/train_ddp.py --model resnet50 --hook ddl --steps 20

Random-init weights and synthetic images/labels (no datasets); per-rank batch fixed (weak
scaling).  Prints one JSON line from rank 0: ms per step (max over ranks, CUDA events),
images/s for the whole job, and the hook used.  Scaling efficiency vs 1 GPU is the SPEC's
100 * t1 / (tN * ... ) arithmetic done by the caller over several N.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from torch.nn.parallel import DistributedDataParallel as DDP  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--hook", default="ddl", choices=["ddl", "nccl"])
    ap.add_argument("--dims", default=None)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world,
                            init_method=None if "MASTER_ADDR" in os.environ else "tcp://127.0.0.1:29533")
    import torchvision
    model = getattr(torchvision.models, a.model)(num_classes=1000).cuda().to(memory_format=torch.channels_last)
    ddp = DDP(model, device_ids=[local], bucket_cap_mb=25, gradient_as_bucket_view=True)
    if a.hook == "ddl":
        from paper_1811_12174_b200 import ddl
        from paper_1811_12174_b200.ddp import ddl_allreduce_hook
        comm = ddl.init(a.dims or {1: "1", 2: "2", 4: "2x2", 8: "2x4"}.get(world, str(world)), max_bytes=64 << 20)
        ddp.register_comm_hook(comm, ddl_allreduce_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.01, momentum=0.9)
    x = torch.randn(a.batch, 3, 224, 224, device="cuda").to(memory_format=torch.channels_last)
    y = torch.randint(0, 1000, (a.batch,), device="cuda")

    def step():
        opt.zero_grad(set_to_none=True)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = torch.nn.functional.cross_entropy(ddp(x), y)
        loss.backward()
        opt.step()

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / a.steps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"model": a.model, "hook": a.hook, "n_gpus": world, "batch_per_gpu": a.batch,
                          "ms_per_step": t.item(), "images_per_s": world * a.batch / (t.item() * 1e-3)}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
