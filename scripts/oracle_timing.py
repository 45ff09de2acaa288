"""Oracle timing on the host cores (SURVEY 8(d) "Oracle timing"): config 1 (P=4, dims 2x2,
1M-element int32 and fp32) and the config-5 sweep points at P=8 up to 256 MiB, for dims
8 / 2x4 / 2x2x2, plus the naive rank-by-rank sum.  A reported baseline, not a target.

  python scripts/oracle_timing.py [--max-bytes 268435456] [--out profiles/r01_oracle_timing.csv]

Columns: what,P,dims,dtype,bytes,s_per_call,busbw_GBs,cores.  busbw = S*2(P-1)/P / t, the
same formula as the GPU rows; numpy elementwise adds run on one core."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synthetic_inputs as si  # noqa: E402


def timed(fn, min_s=0.5):
    fn()  # warm
    k, t0 = 0, time.perf_counter()
    while True:
        fn()
        k += 1
        t = time.perf_counter() - t0
        if t >= min_s:
            return t / k


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-bytes", type=int, default=256 << 20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = ["what,P,dims,dtype,bytes,s_per_call,busbw_GBs,cores"]
    cores = len(os.sched_getaffinity(0))

    def add(what, P, spec, dtype, S, t):
        rows.append(f"{what},{P},{spec},{dtype},{S},{t:.6f},{S * 2 * (P - 1) / P / t / 1e9:.4f},1 (of {cores})")
        print(rows[-1], flush=True)

    # config 1: P = 4, dims 2x2, 1M elements, int32 and fp32, sum; checked vs naive
    for dtype, kind in (("int32", "fullrange"), ("float32", "normal")):
        n = 1 << 20
        bufs = si.rank_buffers(dtype, kind, n, 4)
        dims = oracle.parse_dims("2x2")
        add("oracle-allreduce", 4, "2x2", dtype, 4 * n, timed(lambda: oracle.allreduce(bufs, dims, dtype, "sum")))
        add("naive-sum", 4, "-", dtype, 4 * n, timed(lambda: oracle.naive_sum(bufs, dtype)))
    # config 5 points at P = 8
    S = 1024
    while S <= a.max_bytes:
        n = S // 4
        bufs = si.rank_buffers("float32", "normal", n, 8)
        for spec in ("8", "2x4", "2x2x2"):
            dims = oracle.parse_dims(spec)
            add("oracle-allreduce", 8, spec, "float32", S,
                timed(lambda: oracle.allreduce(bufs, dims, "float32", "sum"), 0.5 if S < (64 << 20) else 0.0))
        add("naive-sum", 8, "-", "float32", S, timed(lambda: oracle.naive_sum(bufs, "float32"), 0.2))
        del bufs
        S *= 16 if S < (1 << 20) else 4
    if a.out:
        with open(a.out, "w") as f:
            f.write("# scripts/oracle_timing.py on the GPU box's host (numpy, 1 core)\n" + "\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
