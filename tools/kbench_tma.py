"""TMA streaming-read sweep (stages x tile bytes x warps/CTA x CTAs/SM)."""
import ctypes
import os
import sys

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


for stages, tileb in ((2, 4096), (3, 4096), (4, 4096), (2, 8192), (3, 8192), (2, 16384), (4, 2048), (8, 2048)):
    for warps, cps in ((4, 5), (4, 4), (8, 2), (8, 3), (2, 8), (1, 16)):
        smem = warps * stages * tileb
        if smem * cps > 220_000:
            continue
        r = timeit(lambda i: lib.kb_tma_read(ctypes.c_void_p(bufs[i % 4].data_ptr()), ctypes.c_int64(n),
                                             ctypes.c_void_p(out.data_ptr()), stages, tileb, warps, cps, sms, st))
        print(f"stages={stages} tile={tileb} warps={warps} ctas/sm={cps} inflight/SM={smem*cps//1024}KB -> {r}")
