"""Experiment: the bench step (ResNet-50 gradient set, 5 buckets, 8 virtual ranks, 2x4, avg)
with buckets all-reduced CONCURRENTLY on K streams by K loopback communicators, each limited
to a share of the CTAs (DDL_CTAS), against the default (one communicator, all CTAs, buckets
back to back).  Question: does overlapping one bucket's L2-bound phases / barrier waits with
another bucket's DRAM-bound phases beat running each bucket on the whole GPU?
  python scripts/concurrent_buckets.py --streams 1,2,3 --ctas 37,18,12"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_12174_b200 import ddl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--streams", default="1,2,3")
ap.add_argument("--ctas", default="37,18,12")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--bucket-events", action="store_true", help="record an event pair around every bucket (as bench.py does)")
ap.add_argument("--grouped", default="", help="also time ddl_group_allreduce_many with these DDL_CHANNELS values, e.g. 1,2,3")
a = ap.parse_args()

P, dims = 8, ddl.parse_dims("2x4")
host = [bench.resnet50_set(r) for r in range(P)]
nb = len(host[0])
dev = torch.device("cuda:0")
bufs = [[torch.from_numpy(host[r][b]).to(dev) for r in range(P)] for b in range(nb)]
main = torch.cuda.current_stream()
for K, C in zip([int(x) for x in a.streams.split(",")], [int(x) for x in a.ctas.split(",")]):
    os.environ["DDL_CTAS"] = str(C)
    comms = [ddl.Loopback(P, dims, device=0) for _ in range(K)]
    os.environ.pop("DDL_CTAS")
    streams = [main] if K == 1 else [torch.cuda.Stream() for _ in range(K)]

    def step():
        for s in streams:
            s.wait_stream(main)
        for b in range(nb):
            if a.bucket_events:
                torch.cuda.Event(enable_timing=True).record(streams[b % K])
            comms[b % K].all_reduce(bufs[b], "avg", stream=streams[b % K])
            if a.bucket_events:
                torch.cuda.Event(enable_timing=True).record(streams[b % K])
        for s in streams:
            main.wait_stream(s)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(a.steps):
        step()
    e1.record(main)
    torch.cuda.synchronize()
    assert all(c.async_error() == 0 for c in comms)
    for b in range(nb):
        assert all(torch.equal(bufs[b][0].view(torch.int32), t.view(torch.int32)) for t in bufs[b][1:])
    ms = e0.elapsed_time(e1) / a.steps
    print(f"streams={K} ctas_cap={C} ctas={[comms[0].ctas_for(h.size, 'float32') for h in host[0]]} "
          f"ms_per_step={ms:.4f}", flush=True)
    for c in comms:
        c.finalize()

for ch in [x for x in a.grouped.split(",") if x]:
    os.environ["DDL_CHANNELS"] = ch
    lb = ddl.Loopback(P, dims, device=0)
    os.environ.pop("DDL_CHANNELS")
    for _ in range(5):
        lb.all_reduce_many(bufs, "avg")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(a.steps):
        lb.all_reduce_many(bufs, "avg")
    e1.record(main)
    torch.cuda.synchronize()
    assert lb.async_error() == 0
    for b in range(nb):
        assert all(torch.equal(bufs[b][0].view(torch.int32), t.view(torch.int32)) for t in bufs[b][1:])
    print(f"grouped channels={ch} ms_per_step={e0.elapsed_time(e1) / a.steps:.4f}", flush=True)
    lb.finalize()
