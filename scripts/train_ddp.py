"""Synthetic synchronous DP-SGD step time (the paper's Table 1 use of DDL), with
DDP's gradient buckets all-reduced by DDL (comm hook) or by NCCL (default).

One configuration (under torchrun):
  torchrun --nproc-per-node N scripts/train_ddp.py --model resnet50|unet3d --hook ddl|nccl --steps 20
prints one JSON line from rank 0: ms per step (max over ranks, CUDA events), samples/s for
the whole job, the hook used.

Table-1 report (plain python; launches the configurations itself):
  python scripts/train_ddp.py --table1 --gpus 1,2,4,8 --model resnet50
prints, per hook, the paper's Table 1 columns (epoch time, speedup w.r.t. previous,
% scaling w.r.t. 1 GPU; paper_1811_12174_b200/report.py) for an epoch of --dataset samples
implied by the weak-scaling step times (per-GPU batch fixed).

Random-init weights and synthetic inputs (no datasets):
* resnet50: torchvision ResNet-50, 224x224 images, 1000 classes (25,557,032 parameters);
* unet3d: the Cicek-layout 3D U-Net of SURVEY.md 8(d) config 3 (19,075,523 parameters in 64
  tensors; conv3^3 + BN + ReLU pairs 3->32->64 | 64->128 | 128->256 | 256->512, transposed
  convs up, skip concatenation, 1x1x1 head to 3 classes), 64^3 volumes (the paper's
  section 4.1 input) -- the paper's own model has no published parameter list.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.nn as nn  # noqa: E402


def _block(i, o):
    return [nn.Conv3d(i, o, 3, padding=1), nn.BatchNorm3d(o), nn.ReLU(inplace=True)]


class UNet3D(nn.Module):
    """Cicek et al. 3D U-Net layout (analysis path doubling channels before each pooling,
    synthesis path with 2x2x2 transposed convolutions and skip concatenation)."""

    def __init__(self, cin=3, ncls=3):
        super().__init__()
        self.e1 = nn.Sequential(*_block(cin, 32), *_block(32, 64))
        self.e2 = nn.Sequential(*_block(64, 64), *_block(64, 128))
        self.e3 = nn.Sequential(*_block(128, 128), *_block(128, 256))
        self.e4 = nn.Sequential(*_block(256, 256), *_block(256, 512))
        self.u3 = nn.ConvTranspose3d(512, 512, 2, stride=2)
        self.d3 = nn.Sequential(*_block(768, 256), *_block(256, 256))
        self.u2 = nn.ConvTranspose3d(256, 256, 2, stride=2)
        self.d2 = nn.Sequential(*_block(384, 128), *_block(128, 128))
        self.u1 = nn.ConvTranspose3d(128, 128, 2, stride=2)
        self.d1 = nn.Sequential(*_block(192, 64), *_block(64, 64))
        self.head = nn.Conv3d(64, ncls, 1)
        self.pool = nn.MaxPool3d(2)

    def forward(self, x):
        s1 = self.e1(x)
        s2 = self.e2(self.pool(s1))
        s3 = self.e3(self.pool(s2))
        b = self.e4(self.pool(s3))
        y = self.d3(torch.cat([self.u3(b), s3], 1))
        y = self.d2(torch.cat([self.u2(y), s2], 1))
        y = self.d1(torch.cat([self.u1(y), s1], 1))
        return self.head(y)


def build(model: str):
    """(module, input shape per sample, loss(out, target), target factory)."""
    if model == "unet3d":
        return UNet3D(), (3, 64, 64, 64), lambda b, dev: torch.randint(0, 3, (b, 64, 64, 64), device=dev)
    import torchvision
    return (torchvision.models.resnet50(num_classes=1000), (3, 224, 224),
            lambda b, dev: torch.randint(0, 1000, (b,), device=dev))


DEFAULT_BATCH = {"resnet50": 64, "unet3d": 2}
DATASET = {"resnet50": 1_281_167, "unet3d": 484}   # ImageNet-1k train; BraTS-2017-size volume count


def run_one(a):
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world,
                            init_method=None if "MASTER_ADDR" in os.environ else "tcp://127.0.0.1:29533")
    net, shape, target = build(a.model)
    cl = torch.channels_last_3d if a.model == "unet3d" else torch.channels_last
    model = net.cuda().to(memory_format=cl)
    ddp = DDP(model, device_ids=[local], bucket_cap_mb=25, gradient_as_bucket_view=True)
    if a.hook == "ddl":
        from paper_1811_12174_b200 import ddl
        from paper_1811_12174_b200.ddp import ddl_allreduce_hook
        comm = ddl.init(a.dims or {1: "1", 2: "2", 4: "2x2", 8: "2x4"}.get(world, str(world)), max_bytes=64 << 20)
        ddp.register_comm_hook(comm, ddl_allreduce_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.01, momentum=0.9)
    b = a.batch or DEFAULT_BATCH[a.model]
    x = torch.randn(b, *shape, device="cuda").to(memory_format=cl)
    y = target(b, "cuda")

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
        print(json.dumps({"model": a.model, "hook": a.hook, "n_gpus": world, "batch_per_gpu": b,
                          "params": sum(p.numel() for p in model.parameters()),
                          "ms_per_step": t.item(), "samples_per_s": world * b / (t.item() * 1e-3)}), flush=True)
    dist.destroy_process_group()


def run_table1(a):
    from paper_1811_12174_b200 import report
    b = a.batch or DEFAULT_BATCH[a.model]
    gpus = [int(x) for x in a.gpus.split(",")]
    res = {}
    for hook in a.hooks.split(","):
        for n in gpus:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                   "--master-addr", "127.0.0.1", "--master-port", str(29540 + n), os.path.abspath(__file__),
                   "--model", a.model, "--hook", hook, "--steps", str(a.steps), "--warmup", str(a.warmup),
                   "--batch", str(b)]
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
            lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            if r.returncode or not lines:
                print(f"# {hook} N={n} failed: {r.stderr[-500:]}", flush=True)
                continue
            d = json.loads(lines[-1])
            print(json.dumps(d), flush=True)
            res.setdefault(hook, {})[n] = d["ms_per_step"]
    for hook, steps in res.items():
        if 1 not in steps:
            continue
        eps = {n: report.epoch_seconds(ms, n, b, a.dataset or DATASET[a.model]) for n, ms in steps.items()}
        print(report.format_rows(report.table1_rows(eps),
                                 f"# Table 1 style: {a.model}, hook {hook}, per-GPU batch {b}, epoch of "
                                 f"{a.dataset or DATASET[a.model]} samples (synthetic, weak-scaling steps)"), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50", choices=["resnet50", "unet3d"])
    ap.add_argument("--hook", default="ddl", choices=["ddl", "nccl"])
    ap.add_argument("--dims", default=None)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--table1", action="store_true", help="launch every (hook, N) and print Table-1 rows")
    ap.add_argument("--gpus", default="1")
    ap.add_argument("--hooks", default="ddl,nccl")
    ap.add_argument("--dataset", type=int, default=0)
    a = ap.parse_args()
    if a.table1:
        run_table1(a)
    else:
        run_one(a)


if __name__ == "__main__":
    main()
