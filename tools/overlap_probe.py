"""Probe: how much of a decode (step i) and the next compress (step i+1) can overlap on one GPU?

Times, with CUDA events over K iterations at the ResNet-50 config (W = 1):
  seq   compress(g_a) then decode(b) on one stream          (today's step structure)
  conc  compress(g_a) on stream 1 || decode(b) on stream 2   (independent buffers)
  c / d each kernel alone
Prints one JSON line.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2110_02140_b200 as s2  # noqa: E402
from paper_2110_02140_b200 import synthetic  # noqa: E402
from paper_2110_02140_b200._lib import S2_MASK_NONZERO, check, lib, ptr  # noqa: E402
from paper_2110_02140_b200.sketch import get_plan  # noqa: E402

# argv: compress density [decode union density] (e.g. 0.01 0.04: a W = 4 step's compress and decode)
cfg = dict(dim=25_600_000, alpha=float(sys.argv[1]) if len(sys.argv) > 1 else 0.01)
cfg["alpha_d"] = float(sys.argv[2]) if len(sys.argv) > 2 else cfg["alpha"]
d, rows, cols = cfg["dim"], 3, 262_144
plan = get_plan(d, d, rows, cols, 0)
gs = [synthetic.gradient(dict(dim=d, alpha=cfg["alpha"] if k < 2 else cfg["alpha_d"], rows=None), 0,
                         base_seed=1234 + 1000 * k) for k in range(4)]
outs = [torch.empty(d, device="cuda") for _ in range(4)]
bms = [torch.empty((d + 31) // 32, dtype=torch.int32, device="cuda") for _ in range(4)]
tabs = [torch.zeros(rows * cols, device="cuda") for _ in range(4)]
cnts = [torch.zeros(4, dtype=torch.int64, device="cuda") for _ in range(4)]
s1, s2_ = torch.cuda.Stream(), torch.cuda.Stream()
import ctypes  # noqa: E402


def comp(k, st):
    check(lib.s2_compress(plan.handle, ptr(gs[k]), ptr(bms[k]), ptr(tabs[k]), S2_MASK_NONZERO, ptr(cnts[k]),
                          ctypes.c_void_p(st.cuda_stream)))


def dec(k, st):
    check(lib.s2_decode(plan.handle, ptr(bms[k]), ptr(tabs[k]), 1, ptr(outs[k]), ctypes.c_void_p(st.cuda_stream)))


for k in range(4):
    comp(k, s1)
torch.cuda.synchronize()
K = 100


def timed(fn):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


cur = torch.cuda.current_stream()
res = {"alpha": cfg["alpha"], "alpha_d": cfg["alpha_d"]}
res["c_us"] = timed(lambda i: comp(i % 2, cur))
res["d_us"] = timed(lambda i: dec(2 + i % 2, cur))
res["seq_us"] = timed(lambda i: (comp(i % 2, cur), dec(2 + i % 2, cur)))


def conc(i):
    s1.wait_stream(cur)
    s2_.wait_stream(cur)
    comp(i % 2, s1)
    dec(2 + i % 2, s2_)
    cur.wait_stream(s1)
    cur.wait_stream(s2_)


res["conc_us"] = timed(conc)
print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in res.items()}))
