"""Drive tools/libkbench.so: read/write pattern sweeps at the ResNet size (experiments)."""
import ctypes
import json
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libkbench.so"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
bufs = [torch.randn(n, device="cuda") * (torch.rand(n, device="cuda") < 0.01) for _ in range(4)]
out = torch.zeros(16, dtype=torch.int32, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def timeit(fn, nbytes, reps=300):
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
    return round(ms * 1e3, 2), round(nbytes / ms / 1e6, 1)


res = {}
for mode in (0, 1, 2):
    for pf in (0, 1):
        for grid in (148 * 2, 148 * 4, 148 * 8, 148 * 16):
            us, gbs = timeit(lambda i: lib.kb_read(ctypes.c_void_p(bufs[i % 4].data_ptr()), ctypes.c_int64(n),
                                                   ctypes.c_void_p(out.data_ptr()), mode, pf, grid, st), 4 * n)
            res[f"read m{mode} pf{pf} g{grid}"] = (us, gbs)
for sh in (0, 1):
    for grid in (148 * 2, 148 * 4, 148 * 8, 148 * 16):
        us, gbs = timeit(lambda i: lib.kb_write(ctypes.c_void_p(bufs[i % 4].data_ptr()), ctypes.c_int64(n), sh,
                                                grid, st), 4 * n)
        res[f"write cs{sh} g{grid}"] = (us, gbs)
for k, v in res.items():
    print(k, v)
print(json.dumps(res))
