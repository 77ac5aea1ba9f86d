"""Isolated kernel loops vs the full step (single GPU): is the step's extra time write-back?"""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2110_02140_b200 import synthetic  # noqa: E402
import paper_2110_02140_b200 as s2  # noqa: E402
from paper_2110_02140_b200._lib import check, lib, ptr  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "resnet50"]
d, rows, cols = cfg["dim"], cfg["rows"], cfg["cols"]
red = s2.S2Reducer(d, rows=rows, cols=cols)
h = red.plan.handle
gs = [synthetic.gradient(dict(dim=d, alpha=cfg["alpha"], rows=cfg.get("grid")), 0, base_seed=1234 + 1000 * k) for k in range(4)]
outs = [torch.empty(d, device="cuda") for _ in range(4)]
tab = torch.zeros(rows * cols + 4, device="cuda")
bm = torch.zeros(-(-d // 32) + 4, dtype=torch.int32, device="cuda")
cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
null = ctypes.c_void_p(0)


def timeit(fn, reps=300):
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 2)


res = {}
res["reduce"] = timeit(lambda i: check(lib.s2_reduce(h, ptr(gs[i % 4]), ptr(outs[i % 4]), null, st)))
res["compress_only(+2 memsets)"] = timeit(lambda i: check(lib.s2_compress(h, ptr(gs[i % 4]), ptr(bm), ptr(tab), 0, ptr(cnt), st)))
check(lib.s2_compress(h, ptr(gs[0]), ptr(bm), ptr(tab), 0, ptr(cnt), st))
res["decode_only"] = timeit(lambda i: check(lib.s2_decode(h, ptr(bm), ptr(tab), 1, ptr(outs[i % 4]), st)))
res["memset_table+counters"] = timeit(lambda i: (tab.zero_(), cnt.zero_()))
print(json.dumps(res))
