"""Small S2 workloads for compute-sanitizer (memcheck / racecheck / synccheck), 1 GPU:
configs[0] (1M / 99 % / 3 x 16384) reduce with element and block bitmaps, the functional
compress/merge/decompress path, block_topk, compaction, and (--local W) the W-rank exchange
on one GPU.  Exits non-zero on a parity failure against the oracle."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_02140_b200 as s2  # noqa: E402
from oracle import s2_oracle as o  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--local", type=int, default=0)
a = ap.parse_args()
d, rows, cols = 1_000_000, 3, 16_384
g = o.synthetic_gradient(d, 0.01, 0, kind="int")
gt = torch.from_numpy(g).cuda()
ref = o.decompress(o.compress(g, g != 0, rows, cols, 0)).astype(np.float32)
if a.local:
    from paper_2110_02140_b200.local import LocalGroup

    grads = [o.synthetic_gradient(d, 0.01, r, kind="int") for r in range(a.local)]
    grp = LocalGroup(a.local, d, rows, cols, timeout_s=60)
    for _ in range(2):
        outs = grp.reduce([torch.from_numpy(x).cuda() for x in grads])
    torch.cuda.synchronize()
    want = o.decompress(o.merge([o.compress(x, x != 0, rows, cols, 0) for x in grads])).astype(np.float32)
    assert all(np.array_equal(x.cpu().numpy(), want) for x in outs), "local exchange parity"
    print("local ok", a.local)
    sys.exit(0)
red = s2.S2Reducer(d, rows=rows, cols=cols)
for _ in range(2):
    out = red.reduce(gt)
red.check()
assert np.array_equal(out.cpu().numpy(), ref)
redb = s2.S2Reducer(d, rows=rows, cols=cols, num_blocks=31_250)
outb = redb.reduce(gt)
p = s2.sparse_compress(gt, None, rows, cols, 0)
q = s2.sparse_compress(gt, None, rows, cols, 0, num_blocks=31_250)
m = s2.sparse_merge([p, p])
assert np.array_equal(s2.sparse_decompress(m).cpu().numpy(), ref)
idx, vals = s2.compacted_values(gt, p.mask)
mk = s2.block_topk(gt, 1000, 50)
_ = s2.sparse_compress(gt, mk, rows, cols, 0)
t = s2.CountSketchTable(5, 1000, 1, d)
t.insert(idx, vals)
_ = t.query(idx)
torch.cuda.synchronize()
print("ok")
