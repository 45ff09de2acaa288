#!/usr/bin/env python
"""Benchmark of the DDL all-reduce (BASELINE.json metric: all-reduce bus GB/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ddl|reference] [--config ...]

One *step* is the whole hot path (every SURVEY.md 8(a) row) over one synchronous-SGD
gradient set: the BASELINE.json configs[1] workload, ResNet-50's 25.6M fp32 gradients in
its 5 DDP buckets, all-reduced with op=avg, dims 2x4 (= [4, 2]).

* N = 1 (no torchrun): LOOPBACK -- the 8 ranks of the 2x4 factorisation are virtual ranks
  on one B200, all in one HBM.  The step runs through the loopback column-chain kernel
  (ddl_chain.cuh: every RS / AG phase of the schedule, per column, in one thread; one launch
  for the 5 buckets); the multi-GPU path's per-CTA slice kernel with device barriers
  (ddl_multi_kernel) is timed on the same step beside it (`slice_kernel`).  Bound: HBM.
* N > 1 (torchrun, one process per GPU): real ranks, peers' buffers mapped over NVLink 5 /
  NVSwitch, dims 8 -> 2x4, 4 -> 2x2, 2 -> 2.  Bound: NVLink.  NCCL's all-reduce on the same
  buffers is timed alongside (comparison only).

value = bus bandwidth = sum_b S_b * 2(P-1)/P / t_step (NCCL-tests convention; per-rank link
bandwidth, the figure the metric's "% of 900 GB/s" refers to).  Timing: W untimed warm-up
steps, then K steps between barrier + synchronize, CUDA events on the launching stream,
max over ranks.  The gradient set (8 x 102 MB) is larger than the 126 MB L2, so no flush
is needed between steps.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


import synthetic_inputs as si  # noqa: E402

METRIC = "allreduce bus GB/s vs msg size at 2/4/8 B200 (% of 900 GB/s NVLink) vs NCCL"
NVLINK_NOMINAL = 900.0
DIMS_FOR_N = {1: "2x4", 2: "2", 4: "2x2", 8: "2x4"}


TRAFFIC_KEY = "resnet50-grad-set 8 virtual ranks dims 2x4 avg, grouped"


def source_hash() -> str:
    """Identity of the kernels a committed ncu capture measured: sha256 of libddl.so's SASS
    (cuobjdump, addresses and encodings stripped) -- so a source edit that compiles to the same
    machine code keeps the capture valid and any kernel change invalidates it; without
    cuobjdump, sha256 of the device sources (.cuh kernel files, planner header, build.sh)."""
    import hashlib
    import re
    lib = os.path.join(ROOT, "paper_1811_12174_b200", "libddl.so")
    side = lib + ".sass-sha"   # written by build.sh right after the build (cuobjdump takes ~10 s)
    try:
        if os.path.getmtime(side) >= os.path.getmtime(lib):
            return open(side).read().strip()
    except OSError:
        pass
    try:
        sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, timeout=120).stdout
        ins = re.findall(r"^\s+/\*[0-9a-f]+\*/\s+(.*?;)", sass, flags=re.M)
        if ins:
            hv = "sass-" + hashlib.sha256("\n".join(ins).encode()).hexdigest()[:16]
            try:
                with open(side, "w") as f:
                    f.write(hv + "\n")
            except OSError:
                pass
            return hv
    except Exception:
        pass
    h = hashlib.sha256()
    src = os.path.join(ROOT, "paper_1811_12174_b200", "csrc")
    for name in sorted(f for f in os.listdir(src) if f.endswith(".cuh")) + ["ddl_plan.h", "../../build.sh"]:
        with open(os.path.join(src, name), "rb") as f:
            h.update(name.encode() + b"\0" + f.read())
    return h.hexdigest()[:16]


def profiled_traffic(workload_key: str):
    """DRAM bytes per step of the timed kernels from the committed ncu capture
    (profiles/traffic.json, written from an `ncu --set full` run of scripts/profile_step.py),
    only if that capture measured THIS build (source hash) and workload -- else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        if d.get("workload") != workload_key or d.get("source_hash") != source_hash():
            return None
        return d["dram_bytes_per_step"]
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- workload
def resnet50_set(rank: int):
    """The gradient set of one rank: 5 DDP buckets (fp32)."""
    return [si.resnet50_bucket(b, rank) for b in range(len(si.resnet50_bucket_bytes()))]


def loopback_hbm_bytes(n: int, P: int, dims, w: int) -> int:
    """Algorithmic HBM bytes of one loopback hierarchical all-reduce (all P virtual ranks):
    per rank, RS phase d reads its g_d group members' copies of the blocks A_{d+1}(r) and
    writes them once; AG phase d reads (g_d - 1)|A_{d+1}| blocks from peers and writes them.
    Exact over ragged block lengths."""
    q = -(-(-(-n // P)) // (16 // w)) * (16 // w)
    blen = [max(0, min(n, (b + 1) * q) - min(n, b * q)) for b in range(P)]
    G = [math.prod(dims[:d]) for d in range(len(dims) + 1)]
    total = 0
    for r in range(P):
        for d, g in enumerate(dims):
            if g == 1:
                continue
            own = [b for b in range(P) if b % G[d + 1] == r % G[d + 1]]            # A_{d+1}(r)
            total += sum(blen[b] for b in own) * (g + 1)                           # RS: g reads + 1 write
            recv = [b for b in range(P) if b % G[d] == r % G[d] and b not in own]  # AG: blocks received
            total += sum(blen[b] for b in recv) * 2                                # read + write
    return total * w


# ----------------------------------------------------------------------------- cpu baseline
def oracle_baseline(P: int, dims, host, budget_s: float = 10.0):
    """The oracle as it stands, on the host cores: whole steps of the same workload (every
    bucket of the gradient set, all P simulated ranks), repeated while under budget_s."""
    import oracle
    nb = len(host[0])
    S = sum(h.size for h in host[0]) * 4
    t0 = time.perf_counter()
    reps = 0
    while True:
        for b in range(nb):
            oracle.allreduce([host[r][b] for r in range(P)], dims, "float32", "avg")
        reps += 1
        el = time.perf_counter() - t0
        if el > budget_s:
            break
    t = el / reps
    return {"value": S * 2 * (P - 1) / P / t / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{reps} whole step(s): the {nb} ResNet-50 buckets ({S} B per rank) x {P} simulated "
                      f"ranks, dims {dims}, avg, {t:.2f} s per step; numpy single-threaded",
            "host_cpus": len(os.sched_getaffinity(0))}


def workload_key(P: int, dims) -> str:
    """The workload both arms name in config.workload (implementation-neutral)."""
    return (f"resnet50-grad-set (25,557,032 fp32 in 5 DDP buckets) all-reduce avg, {P} ranks, dims "
            + "x".join(map(str, dims[::-1])))


def run_reference(args):
    """--impl reference: the oracle (the only 'reference' this paper-only tier has), timed on
    the host cores, each step the whole gradient set of the ddl arm's workload (every bucket,
    all P simulated ranks) -- or, when that would not finish within ~4 minutes for the asked
    --steps/--warmup, one bucket per step (a bounded sample, said in `sample`)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    # the ddl arm's configuration: N = 1 simulates the 8 ranks of 2x4; N > 1 runs N ranks
    P = 8 if args.gpus == 1 else args.gpus
    dims = oracle.parse_dims(args.dims or DIMS_FOR_N.get(args.gpus, str(args.gpus)))
    nb = len(si.resnet50_bucket_bytes())
    host = [[si.resnet50_bucket(b, r) for r in range(P)] for b in range(nb)]   # [bucket][rank]

    def whole():
        for b in range(nb):
            oracle.allreduce(host[b], dims, "float32", "avg")
    t0 = time.perf_counter()
    whole()                                   # first warm-up step, also the estimate
    est = time.perf_counter() - t0
    full = est * (args.steps + args.warmup) <= 240.0
    if full:
        step, nbytes = whole, sum(h[0].size for h in host) * 4
        sample = f"each step: the whole gradient set ({nb} buckets, {nbytes} B per rank) x {P} simulated ranks"
    else:
        step, nbytes = (lambda: oracle.allreduce(host[1], dims, "float32", "avg")), host[1][0].size * 4
        sample = (f"each step: ResNet-50 bucket 1 ({nbytes} B per rank) x {P} simulated ranks (the whole set "
                  f"would take {est:.1f} s per step)")
    for _ in range(max(0, args.warmup - 1)):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    t = (time.perf_counter() - t0) / args.steps
    val = nbytes * 2 * (P - 1) / P / t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_key(P, dims), "dims": "x".join(map(str, dims[::-1])), "n_ranks": P,
                       "ranks": f"{P} simulated ranks in the CPU oracle (numpy, lockstep)",
                       "sample": "whole set" if full else "bucket 1"},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- value gate
def value_gate(lb, sizes, P, dims, dev, bufs, slice_lb=None):
    """Before any timing, the exact step call is checked on VALUES, not only on agreement
    between ranks (a schedule that drops or doubles one rank the same way everywhere would
    still agree):
      1. closed forms through the grouped call on the step's bucket sizes: fp32 x_r = r + 1
         with avg gives (P+1)/2 exactly; int32 x_r[i] = (1<<r) | ((i mod 2^20) << 8) with
         sum gives (2^P - 1) + P * ((i mod 2^20) << 8) mod 2^32 (a missing / doubled rank
         shows in the low byte, a misplaced element in the high bits);
      2. the grouped step on the real gradient set equals the 5 single calls bit for bit
         (the single calls are the path tests/ check element by element against the oracle).
    Restores the buffers to the step's inputs afterwards."""
    import torch
    # 1a. fp32 r+1, avg
    ones = [[torch.full((n,), float(r + 1), device=dev) for r in range(P)] for n in sizes]
    lb.all_reduce_many(ones, "avg")
    # 1b. int32 bitmask, sum
    mask = []
    for n in sizes:
        i = torch.arange(n, device=dev, dtype=torch.int64)
        mask.append([(((i % (1 << 20)) << 8) | (1 << r)).to(torch.int32) for r in range(P)])
    lb.all_reduce_many(mask, "sum")
    torch.cuda.synchronize()
    for b, n in enumerate(sizes):
        assert all(bool((t == (P + 1) / 2).all()) for t in ones[b]), f"closed form r+1 avg failed, bucket {b}"
        i = torch.arange(n, device=dev, dtype=torch.int64)
        want = ((((1 << P) - 1) + P * ((i % (1 << 20)) << 8)) & 0xFFFFFFFF)
        want = torch.where(want >= (1 << 31), want - (1 << 32), want).to(torch.int32)
        assert all(torch.equal(t, want) for t in mask[b]), f"closed form bitmask failed, bucket {b}"
    del ones, mask
    # 2. grouped == single calls, on copies of the step's inputs
    a = [[t.clone() for t in bk] for bk in bufs]
    s_ = [[t.clone() for t in bk] for bk in bufs]
    lb.all_reduce_many(a, "avg")
    for bk in s_:
        lb.all_reduce(bk, "avg")
    torch.cuda.synchronize()
    for b in range(len(sizes)):
        assert all(torch.equal(x.view(torch.int32), y.view(torch.int32)) for x, y in zip(a[b], s_[b])), \
            f"grouped != single calls, bucket {b}"
    # 3. the column-chain kernel == the slice kernels with device barriers (the multi-GPU path's
    #    kernels, DDL_LB_CHAIN=0), bit for bit on the step's inputs
    if slice_lb is not None:
        c_ = [[t.clone() for t in bk] for bk in bufs]
        slice_lb.all_reduce_many(c_, "avg")
        torch.cuda.synchronize()
        for b in range(len(sizes)):
            assert all(torch.equal(x.view(torch.int32), y.view(torch.int32)) for x, y in zip(a[b], c_[b])), \
                f"chain kernel != slice kernel, bucket {b}"
        del c_
    return ("closed forms (fp32 r+1 avg, int32 bitmask sum) through the grouped call on the step's bucket "
            "sizes; grouped step == 5 single calls bitwise; column-chain kernel == barrier slice kernel bitwise; "
            "all ranks identical after warm-up")


# ----------------------------------------------------------------------------- N = 1: loopback
def run_loopback(args):
    import torch
    from paper_1811_12174_b200 import ddl

    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    P = 8
    dims = ddl.parse_dims(args.dims or DIMS_FOR_N[1])
    lb = ddl.Loopback(P, dims, device=0)
    # the same step through the per-CTA slice kernels with device barriers (the kernels the
    # multi-GPU path runs; context, timed after the headline)
    os.environ["DDL_LB_CHAIN"] = "0"
    try:
        slice_lb = ddl.Loopback(P, dims, device=0)
    finally:
        os.environ.pop("DDL_LB_CHAIN", None)
    host = [resnet50_set(r) for r in range(P)]                 # [rank][bucket]
    nb = len(host[0])
    sizes = [h.size for h in host[0]]
    bufs = [[torch.from_numpy(host[r][b]).to(dev) for r in range(P)] for b in range(nb)]   # [bucket][rank]
    S_total = sum(sizes) * 4
    stream = torch.cuda.current_stream()

    # One step = the whole gradient set: the 5 buckets in ONE grouped all-reduce
    # (ddl_group_allreduce_many: each bucket runs the full 2x4 schedule; the buckets share
    # the launch over DDL_CHANNELS channels of CTAs).  Bit-identical to 5 single calls.
    def step():
        lb.all_reduce_many(bufs, "avg")

    def seq_step(evs=None):   # the same set as 5 single calls (context: "sequential")
        for b in range(nb):
            if evs is not None:
                evs[b][0].record(stream)
            lb.all_reduce(bufs[b], "avg")
            if evs is not None:
                evs[b][1].record(stream)

    gate = value_gate(lb, sizes, P, dims, dev, bufs, slice_lb)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:   # sampling spans warm-up + timed region (>= a few 100-ms samples)
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        assert lb.async_error() == ddl.SUCCESS
        for b in range(nb):   # correctness gate: all virtual ranks bit-identical
            assert all(torch.equal(bufs[b][0].view(torch.int32), t.view(torch.int32)) for t in bufs[b][1:])
        t_pad = time.perf_counter()
        while time.perf_counter() - t_pad < 0.3:   # keep the GPU busy so the sampler sees load clocks
            step()
            torch.cuda.synchronize()
        # the timed region: exactly K steps between two events, nothing else on the stream
        t_start.record(stream)
        for k in range(args.steps):
            step()
        t_end.record(stream)
        torch.cuda.synchronize()
        # kernel durations for the roofline: a second pass of K steps with an event pair
        # around every launch (an event between launches costs ~2-3 us of GPU time, so it
        # stays out of the headline region)
        kev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        for k in range(args.steps):
            kev[k][0].record(stream)
            step()
            kev[k][1].record(stream)
        torch.cuda.synchronize()
        # context: the same set as 5 single calls, per-bucket events
        sev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(nb)] for _ in range(args.steps)]
        for k in range(args.steps):
            seq_step(sev[k])
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for k in range(args.steps):
            seq_step()
        s1.record(stream)
        # context: the same grouped step through the slice kernel with device barriers
        for _ in range(2):
            slice_lb.all_reduce_many(bufs, "avg")
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        for k in range(args.steps):
            slice_lb.all_reduce_many(bufs, "avg")
        m1.record(stream)
        torch.cuda.synchronize()
    assert lb.async_error() == ddl.SUCCESS and slice_lb.async_error() == ddl.SUCCESS
    slice_ms = m0.elapsed_time(m1) / args.steps
    ms = t_start.elapsed_time(t_end) / args.steps
    busbw = S_total * 2 * (P - 1) / P / (ms * 1e-3) / 1e9
    kern_ms = sum(kev[k][0].elapsed_time(kev[k][1]) for k in range(args.steps))
    seq_ms = s0.elapsed_time(s1) / args.steps
    bucket_us = [sum(sev[k][b][0].elapsed_time(sev[k][b][1]) for k in range(args.steps)) / args.steps * 1e3
                 for b in range(nb)]
    n_oneshot = sum(1 for s in sizes if lb.algo_for(s, "float32") == ddl.ALGO_ONESHOT)
    launches_per_step = n_oneshot + -(-(nb - n_oneshot) // 8)
    # Roofline numerator: the all-reduce's COMPULSORY HBM bytes in one GPU -- every virtual
    # rank's input read once and its result written once, 2 * P * S per step (as K5's
    # (g+1)*n*w).  The schedule's own phase bytes (27/8 * S per rank for 2x4, many of them
    # L2 hits) are reported beside it; against the copy peak they exceed 1.
    algo_bytes = 2 * P * S_total * args.steps
    sched_bytes = sum(loopback_hbm_bytes(n, P, dims, 4) for n in sizes) * args.steps
    hbm_peak, peak_src = peaks()
    # the kernel's average launch duration: the timed region holds nothing but this kernel's
    # launches (one per step), so the CUDA-event span of the region / launches is it; the
    # second pass's per-launch event pairs (kern_ms) add the launch gap that back-to-back
    # launches hide (programmatic dependent launch) and are reported beside it
    launch_ms = ms * args.steps if launches_per_step == 1 else kern_ms
    achieved = algo_bytes / (launch_ms * 1e-3) / 1e9

    # e2e through the public API with HOST buffers: per step H2D of every rank's buckets from
    # pinned memory, the all-reduce, D2H of the reduced gradient set (identical on all ranks).
    pinned = [[torch.from_numpy(host[r][b]).pin_memory() for r in range(P)] for b in range(nb)]
    out_host = [torch.empty(s, dtype=torch.float32).pin_memory() for s in sizes]
    e2e_steps = max(3, min(args.steps, 10))

    # pipelined like a user would: bucket b's H2D (copy stream) overlaps bucket b-1's
    # all-reduce (compute stream) and bucket b-2's D2H (second copy stream)
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_step():
        for b in range(nb):
            with torch.cuda.stream(h2d_s):
                for r in range(P):
                    bufs[b][r].copy_(pinned[b][r], non_blocking=True)
            stream.wait_stream(h2d_s)
            lb.all_reduce(bufs[b], "avg", stream=stream)
            d2h_s.wait_stream(stream)
            with torch.cuda.stream(d2h_s):
                out_host[b].copy_(bufs[b][0], non_blocking=True)
        stream.wait_stream(d2h_s)
        h2d_s.wait_stream(stream)   # the next step's H2D must not overwrite buffers still in use

    e2e_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h2d_s.wait_stream(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps

    # K5: local reduce/scale, g = 8 fp32 buffers of 64 MiB -> out, vs HBM
    g, n5 = 8, (64 << 20) // 4
    ins = [torch.randn(n5, device=dev) for _ in range(g)]
    out5 = torch.empty(n5, device=dev)
    for _ in range(3):
        ddl.local_reduce(ins, out5, 1.0 / g)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    k0.record(stream)
    reps5 = 20
    for _ in range(reps5):
        ddl.local_reduce(ins, out5, 1.0 / g)
    k1.record(stream)
    torch.cuda.synchronize()
    k5_ms = k0.elapsed_time(k1) / reps5
    k5_gbs = (g + 1) * n5 * 4 / (k5_ms * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": busbw, "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_key(P, dims),
                   "ranks": "8 virtual ranks on one B200 (loopback: the column-chain kernel runs every phase "
                            "of the schedule per column in one thread)",
                   "dims": "x".join(map(str, dims[::-1])), "n_ranks": P, "bytes_per_rank": S_total,
                   "buckets": sizes, "l2": "inputs (8 x 102 MB) larger than L2, no flush",
                   "algo": ["oneshot" if lb.algo_for(s, "float32") == ddl.ALGO_ONESHOT else "hier" for s in sizes],
                   "step": "one grouped all-reduce of the 5 buckets (ddl_group_allreduce_many, column-chain "
                           f"kernel, {launches_per_step} launch(es))",
                   "slice_kernel": {"ms_per_step": round(slice_ms, 4),
                                    "value": S_total * 2 * (P - 1) / P / (slice_ms * 1e-3) / 1e9,
                                    "frac": 2 * P * S_total / (slice_ms * 1e-3) / 1e9 / hbm_peak,
                                    "kernel": "ddl_multi_kernel<float> (the multi-GPU path's per-CTA slice "
                                              "kernel with device barriers, DDL_LB_CHAIN=0; same step, "
                                              "bit-identical results, checked in the gate)"},
                   "sequential": {"ms_per_step": round(seq_ms, 4), "calls": "5 single ddl_group_allreduce",
                                  "ctas_per_rank": [lb.ctas_for(s, "float32") for s in sizes],
                                  "bucket_us": [round(u, 1) for u in bucket_us]}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak,
                     "traffic": (tr // launches_per_step if (tr := profiled_traffic(TRAFFIC_KEY))
                                 and dims == [4, 2] else None),
                     "traffic_unit": "DRAM bytes per launch, ncu --set full of one bench step, profiles/traffic.json "
                                     "(null unless that capture measured this build: source hash)",
                     "algorithmic_bytes_per_launch": algo_bytes // args.steps // launches_per_step,
                     "peak_source": peak_src,
                     "kernel": "ddl_chain_tma_kernel<float, CT<2,4,2>> (loopback column chain: 5 buckets x 8 "
                               "virtual ranks in one launch, every RS/AG phase per column in one thread, "
                               "first-phase sources staged by TMA bulk copies)",
                     "kernel_timing": ("CUDA events over the timed region, one launch per step (region / K)"
                                       if launches_per_step == 1 else
                                       "second pass of K steps, CUDA events around every launch"),
                     "per_launch_events_ms": kern_ms / args.steps,
                     "algorithmic_bytes": "compulsory: 2 x 8 virtual ranks x 102,228,128 B per step "
                                          "(each input read once, each result written once)",
                     "algorithmic_bytes_per_step": algo_bytes // args.steps,
                     "schedule_bytes_per_step": sched_bytes // args.steps,
                     "schedule_frac": sched_bytes / (launch_ms * 1e-3) / 1e9 / hbm_peak,
                     "kernel_ms_per_step": launch_ms / args.steps,
                     # physical view: profiled DRAM bytes of a step / this run's kernel time
                     "dram_frac": ((tr2 / (launch_ms / args.steps * 1e-3) / 1e9 / hbm_peak)
                                   if (tr2 := profiled_traffic(TRAFFIC_KEY)) and dims == [4, 2] else None)},
        "e2e": {"value": S_total * 2 * (P - 1) / P / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": S_total * P, "d2h_bytes_per_step": S_total,
                "how": "per bucket, pipelined on three streams: pinned H2D of the 8 ranks' copies || "
                       "ddl_group_allreduce || D2H of the reduced bucket (PCIe-bound)"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
        "correctness_gate": gate,
        "local_reduce": {"g": g, "bytes": (g + 1) * n5 * 4, "ms": k5_ms, "achieved": k5_gbs, "peak": hbm_peak,
                         "unit": "GB/s", "frac": k5_gbs / hbm_peak},
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = oracle_baseline(P, dims, host)
    print(json.dumps(line), flush=True)
    lb.finalize()
    slice_lb.finalize()


# ----------------------------------------------------------------------------- N > 1
def peer_copy_gbs(comm, P, rank, nbytes, offset, reps=10):
    """Peer-copy peak measured in the same run: every rank copies nbytes from its own
    symmetric buffer into rank (r+1) mod P's (mapped over NVLink), all ranks at once
    (cudaMemcpyAsync on UVA peer pointers = the copy engines), so each GPU sends and
    receives one stream: GB/s per direction per GPU, max time over ranks."""
    import torch
    import torch.distributed as dist
    peer, dst_off = (rank + 1) % P, offset + (nbytes + 255) // 256 * 256
    stream = torch.cuda.current_stream()
    for _ in range(2):
        comm.peer_copy(peer, offset, dst_off, nbytes, stream)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        comm.peer_copy(peer, offset, dst_off, nbytes, stream)
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    return nbytes / (t.item() * 1e-3) / 1e9


def run_multi(args):
    import torch
    import torch.distributed as dist
    from paper_1811_12174_b200 import ddl

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    # DDL_BENCH_SAME_GPU=1: functional check of this code path with every rank on cuda:0
    # (gloo bootstrap, no NCCL comparison; the kernels are time-sliced -- numbers meaningless)
    same_gpu = os.environ.get("DDL_BENCH_SAME_GPU") == "1"
    dev_idx = 0 if same_gpu else local
    torch.cuda.set_device(dev_idx)
    if same_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
    P = world
    dims = ddl.parse_dims(args.dims or DIMS_FOR_N.get(P, str(P)))
    host = resnet50_set(rank)
    sizes = [h.size for h in host]
    S_total = sum(sizes) * 4
    copy_bytes = 64 << 20
    sym_bytes = (S_total + 256 * len(sizes) + 255) // 256 * 256
    comm = ddl.init(dims, max_bytes=sym_bytes + 2 * copy_bytes + (1 << 20))
    offs, views = 0, []
    for h in host:                                   # buckets live in the symmetric buffer (zero-copy)
        v = comm.buffer(h.size, torch.float32, offs)
        v.copy_(torch.from_numpy(h))
        views.append(v)
        offs += (h.size * 4 + 255) // 256 * 256
    stream = torch.cuda.current_stream()
    cuda_or_cpu = "cpu" if same_gpu else "cuda"

    def step():   # the 5 buckets in one grouped all-reduce (as at N = 1)
        comm.all_reduce_many(views, "avg")

    # A rank's 102 MB gradient set fits its 126 MB L2, so between timed steps every rank
    # overwrites a 256 MiB buffer (outside the events): each step reads its buckets, and
    # its peers' buckets over NVLink, from HBM.
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev_idx}")

    def timed(fn, steps, flush=True):
        torch.cuda.synchronize()
        dist.barrier()
        evs = []
        for _ in range(steps):
            if flush:
                l2_flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([sum(a.elapsed_time(b) for a, b in evs) / steps], device=cuda_or_cpu)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)   # max over ranks
        return t.item()

    # correctness gate on values before any timing: closed forms through the grouped call
    # (fp32 r+1 avg -> (P+1)/2 exactly; int32 bitmask sum -> (2^P-1) + P*((i mod 2^20)<<8))
    gate_ok = True
    for kind in ("r+1", "bitmask"):
        o2, tv = 0, []
        for n in sizes:
            t = comm.buffer(n, torch.float32 if kind == "r+1" else torch.int32, o2)
            if kind == "r+1":
                t.fill_(float(rank + 1))
            else:
                i = torch.arange(n, device=f"cuda:{dev_idx}", dtype=torch.int64)
                t.copy_((((i % (1 << 20)) << 8) | (1 << rank)).to(torch.int32))
            tv.append(t)
            o2 += (n * 4 + 255) // 256 * 256
        comm.all_reduce_many(tv, "avg" if kind == "r+1" else "sum")
        torch.cuda.synchronize()
        for t, n in zip(tv, sizes):
            if kind == "r+1":
                gate_ok &= bool((t == (P + 1) / 2).all())
            else:
                i = torch.arange(n, device=f"cuda:{dev_idx}", dtype=torch.int64)
                w_ = (((1 << P) - 1) + P * ((i % (1 << 20)) << 8)) & 0xFFFFFFFF
                gate_ok &= torch.equal(t, torch.where(w_ >= (1 << 31), w_ - (1 << 32), w_).to(torch.int32))
    okt = torch.tensor([0 if gate_ok else 1], device=cuda_or_cpu)
    dist.all_reduce(okt, op=dist.ReduceOp.MAX)
    assert okt.item() == 0, "closed-form gate failed on some rank"
    for v, h in zip(views, host):                     # restore the gradient set
        v.copy_(torch.from_numpy(h))

    for _ in range(args.warmup):
        step()
    # all ranks bit-identical after the warm-up steps
    digest = torch.tensor([int(v.view(torch.int32).to(torch.int64).sum().item()) for v in views], dtype=torch.int64)
    alld = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(alld, digest.cuda() if not same_gpu else digest)
    assert all(torch.equal(d.cpu(), alld[0].cpu()) for d in alld), "ranks disagree after all-reduce"
    with ClockSampler(dev_idx) as clk:
        ms = timed(step, args.steps)
    assert comm.async_error() == ddl.SUCCESS
    busbw = S_total * 2 * (P - 1) / P / (ms * 1e-3) / 1e9
    singles = sum(1 for s in sizes if comm.algo_for(s, "float32") != ddl.ALGO_HIER)
    launches = singles + -(-(len(sizes) - singles) // 8)

    # per-bucket bus bandwidth: each bucket as one single call (events per call, max over ranks)
    per_bucket = []
    for v, n in zip(views, sizes):
        tb = timed(lambda v=v: comm.all_reduce(v, "avg"), max(3, min(args.steps, 20)))
        per_bucket.append({"bytes": n * 4, "us": round(tb * 1e3, 2),
                           "busbw": round(n * 4 * 2 * (P - 1) / P / (tb * 1e-3) / 1e9, 1)})

    # peer-copy peak of this box, measured now (the roofline's measured denominator)
    peer_gbs = peer_copy_gbs(comm, P, rank, copy_bytes, sym_bytes)

    nccl = None
    if not same_gpu:
        nccl = {"version": ".".join(map(str, torch.cuda.nccl.version()))}
        nccl_bufs = [torch.from_numpy(h).cuda() for h in host]

        def nccl_step(group=None):
            for t in nccl_bufs:
                dist.all_reduce(t, op=dist.ReduceOp.AVG, group=group)
        for _ in range(args.warmup):
            nccl_step()
        nccl_ms = timed(nccl_step, args.steps)
        nccl["default"] = {"value": S_total * 2 * (P - 1) / P / (nccl_ms * 1e-3) / 1e9, "unit": "GB/s",
                           "ms_per_step": nccl_ms}
        # NCCL with its NVLS (NVSwitch multicast) algorithms excluded: a second communicator
        # created while NCCL_ALGO excludes them (NCCL reads NCCL_ALGO at communicator init;
        # NCCL_NVLS_ENABLE is cached per process, so it cannot be toggled here)
        old = os.environ.get("NCCL_ALGO")
        try:
            os.environ["NCCL_ALGO"] = "^NVLS,NVLSTree"
            g2 = dist.new_group(list(range(world)))
            for _ in range(args.warmup):
                nccl_step(g2)
            t2 = timed(lambda: nccl_step(g2), args.steps)
            nccl["no_nvls"] = {"value": S_total * 2 * (P - 1) / P / (t2 * 1e-3) / 1e9, "unit": "GB/s",
                               "ms_per_step": t2, "how": "NCCL_ALGO=^NVLS,NVLSTree on a second communicator"}
        except Exception as e:   # record, never fail the bench line on the comparison
            nccl["no_nvls"] = {"error": repr(e)[:200]}
        finally:
            if old is None:
                os.environ.pop("NCCL_ALGO", None)
            else:
                os.environ["NCCL_ALGO"] = old

    # e2e: host gradients -> device (pinned H2D), all-reduce, reduced gradients -> host
    pinned = [torch.from_numpy(h).pin_memory() for h in host]
    outh = [torch.empty(s).pin_memory() for s in sizes]

    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_step():   # pipelined: H2D of bucket b || all-reduce of b-1 || D2H of b-2
        for v, ph, oh in zip(views, pinned, outh):
            with torch.cuda.stream(h2d_s):
                v.copy_(ph, non_blocking=True)
            stream.wait_stream(h2d_s)
            comm.all_reduce(v, "avg", stream=stream)
            d2h_s.wait_stream(stream)
            with torch.cuda.stream(d2h_s):
                oh.copy_(v, non_blocking=True)
        stream.wait_stream(d2h_s)
        h2d_s.wait_stream(stream)
    e2e_step()
    e2e_ms = timed(e2e_step, max(3, min(args.steps, 10)), flush=False)   # fresh H2D data every step

    # the oracle on the same per-rank set at P simulated ranks (rank 0 only, bounded)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = oracle_baseline(P, dims, [resnet50_set(r) for r in range(P)])
    dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": busbw, "unit": "GB/s", "n_gpus": P, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_key(P, dims), "ranks": f"{P} ranks, one per GPU",
                       "dims": "x".join(map(str, dims[::-1])), "n_ranks": P, "bytes_per_rank": S_total,
                       "buckets": sizes, "same_gpu": same_gpu,
                       "step": "one grouped all-reduce of the 5 buckets (ddl_allreduce_many, zero-copy buffers)",
                       "l2": "flushed between timed steps (256 MiB write per rank, outside the per-step events)"},
            # roofline: NVLink per direction per GPU; algorithmic bytes 2S(P-1)/P for every
            # factorisation, so `achieved` = the bus bandwidth
            "roofline": {"bound": "nvlink", "achieved": busbw, "peak": NVLINK_NOMINAL, "unit": "GB/s",
                         "frac": busbw / NVLINK_NOMINAL,
                         "peak_source": "north_star: 900 GB/s per direction per GPU (NVLink 5 nominal)",
                         "measured_peer_copy": peer_gbs,
                         "frac_of_measured_peer_copy": busbw / peer_gbs if peer_gbs else None,
                         "peer_copy_how": f"all ranks at once, {copy_bytes} B own buffer -> rank+1's "
                                          "(cudaMemcpyAsync over the cudaIpc mapping), max over ranks",
                         "algorithmic_bytes_per_step": int(S_total * 2 * (P - 1) / P),
                         "traffic": None,
                         "traffic_how": "NVLink bytes need ncu with --replay-mode application on every rank: "
                                        "scripts/ncu_nvlink.sh"},
            "per_bucket": per_bucket,
            "nccl": nccl,
            "e2e": {"value": S_total * 2 * (P - 1) / P / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": S_total, "d2h_bytes_per_step": S_total},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "correctness_gate": "closed forms (fp32 r+1 avg, int32 bitmask sum) through the grouped call on "
                                "the step's bucket sizes, every rank; all ranks identical after warm-up",
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    comm.finalize()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ddl", choices=["ddl", "reference"])
    ap.add_argument("--dims", default=None, help="override the factorisation, e.g. 2x2x2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_multi(args)
    else:
        run_loopback(args)


if __name__ == "__main__":
    main()
