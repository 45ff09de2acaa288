"""Is the loopback chain kernel's time sensitive to where the virtual ranks' buffers sit?
The bench step (ResNet-50 set, 8 virtual ranks, 2x4, avg, grouped) timed by CUDA-graph replay
with the same data in several placements: one tensor per (bucket, rank) allocated bucket-major
(step_ab.py's layout) or rank-major, every rank's buckets packed in one tensor, and packed with
a pad of 1-15 x 4 KiB between ranks.  Run under DDL_LIB / DDL_* like step_ab.py."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_12174_b200 import ddl  # noqa: E402


def timeit(lb, bufs, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                lb.all_reduce_many(bufs, "avg")
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    del g
    return statistics.median(ts)


def main():
    P = 8
    host = [bench.resnet50_set(r) for r in range(P)]
    nb = len(host[0])
    sizes = [h.size for h in host[0]]
    lb = ddl.Loopback(P, ddl.parse_dims("2x4"))
    layouts = {}
    layouts["bucket-major"] = lambda: [[torch.from_numpy(host[r][b]).cuda() for r in range(P)] for b in range(nb)]

    def rank_major():
        t = [[torch.from_numpy(host[r][b]).cuda() for b in range(nb)] for r in range(P)]
        return [[t[r][b] for r in range(P)] for b in range(nb)]
    layouts["rank-major"] = rank_major

    def packed(pad_pages):
        def f():
            tot = sum((n + 63) // 64 * 64 for n in sizes)
            out = [[None] * P for _ in range(nb)]
            for r in range(P):
                big = torch.empty(tot + pad_pages * r * 1024 + 1024, device="cuda")
                off = pad_pages * r * 1024
                for b in range(nb):
                    v = big[off:off + sizes[b]]
                    v.copy_(torch.from_numpy(host[r][b]))
                    out[b][r] = v
                    off += (sizes[b] + 63) // 64 * 64
            return out
        return f
    layouts["packed"] = packed(0)
    for pp in (1, 3, 7, 15):
        layouts[f"packed+{pp}x4KiB*r"] = packed(pp)
    for name, mk in layouts.items():
        bufs = mk()
        t = timeit(lb, bufs)
        addr = [bufs[1][r].data_ptr() for r in range(P)]
        d = [(a - addr[0]) for a in addr]
        print(f"{name:22s} ms/step {t:.4f}   bucket-1 rank offsets (MiB) {[round(x / 2**20, 3) for x in d]}", flush=True)
        del bufs
        torch.cuda.empty_cache()
    lb.finalize()


if __name__ == "__main__":
    main()
