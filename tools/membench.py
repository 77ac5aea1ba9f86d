"""Practical memory rooflines on this B200 for the access patterns of the S2 kernels:
read-only stream (sum), write-only stream (fill), and copy, at the ResNet config size."""
import json
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
bufs = [torch.randn(n, device="cuda") for _ in range(4)]
outs = [torch.empty(n, device="cuda") for _ in range(4)]
res = {}


def timeit(fn, nbytes, reps=200):
    for i in range(10):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"us": round(ms * 1e3, 2), "GB/s": round(nbytes / ms / 1e6, 1)}


acc = torch.empty((), device="cuda")
res["read_sum"] = timeit(lambda i: torch.sum(bufs[i % 4], dim=0, out=acc), 4 * n)
res["write_fill"] = timeit(lambda i: outs[i % 4].fill_(0.0), 4 * n)
res["copy"] = timeit(lambda i: outs[i % 4].copy_(bufs[i % 4]), 8 * n)
res["memset"] = timeit(lambda i: outs[i % 4].zero_(), 4 * n)
print(json.dumps({"n": n, **res}))
