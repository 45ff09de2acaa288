"""Write synthetic_inputs/resnet50_buckets.json: ResNet-50's parameter tensors grouped
into the DDP gradient buckets (first bucket 1 MiB cap, then 25 MiB, reversed order) that
BASELINE.json config 2 names.  Shapes only -- no weights; torchvision is used once, here,
so the GPU box does not need it.  Run: python scripts/gen_resnet50_buckets.py
"""
import json, math, os
import torch.distributed as dist
import torchvision

m = torchvision.models.resnet50()
named = list(m.named_parameters())[::-1]        # DDP assigns buckets over reversed params
params = [p for _, p in named]
assign = dist._compute_bucket_assignment_by_size(params, [1 << 20, 25 << 20], [False] * len(params))[0]
buckets = []
for idx in assign:
    tensors = []
    for i in idx:
        name, p = named[i]
        shape = list(p.shape)
        fan_in = math.prod(shape[1:]) if len(shape) > 1 else shape[0]
        tensors.append({"name": name, "shape": shape, "numel": p.numel(), "fan_in": fan_in})
    buckets.append({"bytes": 4 * sum(t["numel"] for t in tensors), "tensors": tensors})
out = os.path.join(os.path.dirname(__file__), "..", "synthetic_inputs", "resnet50_buckets.json")
with open(out, "w") as f:
    json.dump({"model": "torchvision resnet50", "total_params": sum(p.numel() for p in params),
               "buckets": buckets}, f, indent=0)
print([b["bytes"] for b in buckets])
