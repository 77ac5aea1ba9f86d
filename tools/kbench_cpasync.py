"""cp.async ring streaming-read sweep vs the LDG pattern (experiment)."""
import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libkbench.so"))
n = 25_600_000
bufs = [torch.randn(n, device="cuda") for _ in range(4)]
out = torch.zeros(16, dtype=torch.int32, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
sms = torch.cuda.get_device_properties(0).multi_processor_count


def timeit(fn, reps=200):
    for i in range(5):
        assert fn(i) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return round(ms * 1e3, 2), round(4 * n / ms / 1e6, 1)


for stages in (2, 3, 4):
    for warps, cps in ((4, 4), (4, 6), (8, 2), (8, 3), (4, 8), (2, 12)):
        if warps * stages * 4096 * cps > 220_000:
            continue
        r = timeit(lambda i: lib.kb_cpasync_read(ctypes.c_void_p(bufs[i % 4].data_ptr()), ctypes.c_int64(n),
                                                 ctypes.c_void_p(out.data_ptr()), stages, warps, cps, sms, st))
        print(f"cpasync stages={stages} warps={warps} ctas/sm={cps} -> {r}")
for grid in (148 * 2, 148 * 4, 148 * 8, 148 * 16):
    r = timeit(lambda i: lib.kb_read(ctypes.c_void_p(bufs[i % 4].data_ptr()), ctypes.c_int64(n),
                                     ctypes.c_void_p(out.data_ptr()), 0, 1, grid, st))
    print(f"ldg prefetch grid={grid} -> {r}")
