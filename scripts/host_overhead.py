"""Host cost per call (CPU wall time of N asynchronous calls, tiny message so the GPU keeps
up): the Python wrapper vs a raw ctypes call with prebuilt arguments, loopback
(cooperative launch) vs one in-process rank (plain launch)."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_12174_b200 import ddl

N = 2000
L = ddl.lib()


def per_call(fn, n=N):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    el = time.perf_counter() - t
    torch.cuda.synchronize()
    return el / n * 1e6


lb = ddl.Loopback(8, [4, 2])
bufs = [torch.ones(256, device="cuda") for _ in range(8)]
ptrs = ddl._ptrs([b.data_ptr() for b in bufs])
s = torch.cuda.current_stream().cuda_stream
print(f"loopback wrapper      {per_call(lambda: lb.all_reduce(bufs)):.2f} us/call")
print(f"loopback raw ctypes   {per_call(lambda: L.ddl_group_allreduce(lb.h, ptrs, 256, ddl.FLOAT32, ddl.SUM, s)):.2f} us/call")
x = torch.ones(256, device="cuda")
print(f"torch x.add_(1)       {per_call(lambda: x.add_(1)):.2f} us/call")
print(f"current_stream()      {per_call(lambda: torch.cuda.current_stream().cuda_stream):.2f} us/call")
print(f"local_reduce g=2      {per_call(lambda: ddl.local_reduce([x, x], x)):.2f} us/call")
lb.finalize()
