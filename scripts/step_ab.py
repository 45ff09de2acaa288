"""A/B of the bench step (N = 1: ResNet-50 gradient set, 8 virtual ranks, 2x4, avg, one
grouped call) under DDL_* settings read at Loopback init.  Each configuration: value check
(grouped == 5 single calls, bitwise), then CUDA-graph replay of 20 steps, median of 5
trials (ms per step).  With --ncu the script instead runs ONE configuration for W + 1
steps (profile target: ncu -k regex:ddl_multi -s W -c 1 --metrics dram__bytes_read.sum,...).

  python scripts/step_ab.py 'DDL_CHANNELS=2' 'DDL_CHANNELS=2,DDL_GROUP_WAVE_MB=32' ...
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_12174_b200 import ddl  # noqa: E402


def parse(cfg):
    return dict(kv.split("=") for kv in cfg.split(",") if kv)


def make_lb(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return ddl.Loopback(8, ddl.parse_dims(os.environ.get("AB_DIMS", "2x4")))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    ncu = "--ncu" in sys.argv
    P = 8
    host = [bench.resnet50_set(r) for r in range(P)]
    nb = len(host[0])
    bufs = [[torch.from_numpy(host[r][b]).cuda() for r in range(P)] for b in range(nb)]
    ref = None
    for cfg in args or [""]:
        lb = make_lb(parse(cfg))
        if ncu:
            for _ in range(4):
                lb.all_reduce_many(bufs, "avg")
            torch.cuda.synchronize()
            return
        a = [[t.clone() for t in bk] for bk in bufs]
        lb.all_reduce_many(a, "avg")
        torch.cuda.synchronize()
        if ref is None:
            ref = [[t.clone() for t in bk] for bk in bufs]
            for bk in ref:
                lb.all_reduce(bk, "avg")
            torch.cuda.synchronize()
        ok = all(torch.equal(x.view(torch.int32), y.view(torch.int32)) for bx, by in zip(a, ref) for x, y in zip(bx, by))
        del a
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
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
            ts.append(e0.elapsed_time(e1) / 20)
        # value check again after the timed calls (learned state, if any, now in use)
        a = [[t.clone() for t in bk] for bk in bufs]
        lb.all_reduce_many(a, "avg")
        torch.cuda.synchronize()
        ok2 = all(torch.equal(x.view(torch.int32), y.view(torch.int32)) for bx, by in zip(a, ref) for x, y in zip(bx, by))
        del a
        print(f"{cfg or 'default':60s} ms/step {statistics.median(ts):.4f} (min {min(ts):.4f}) ok={ok} ok_after={ok2} "
              f"err={lb.async_error()}", flush=True)
        del g
        lb.finalize()


if __name__ == "__main__":
    main()
