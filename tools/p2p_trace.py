"""Per-phase timing of the peer-memory exchange kernel from in-kernel globaltimer stamps.

    S2_P2P_TRACE=1 torchrun --nproc-per-node N tools/p2p_trace.py
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import s2_oracle as o  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
import paper_2110_02140_b200 as s2  # noqa: E402
from paper_2110_02140_b200._lib import check, lib  # noqa: E402

d = 25_600_000
red = s2.S2Reducer(d, rows=3, cols=262144)
g = torch.from_numpy(o.synthetic_gradient(d, 0.01, rank)).cuda()
out = torch.empty(d, device="cuda")
res = []
for it in range(30):
    for _ in range(8):  # back-to-back (no host sync between reduces): steady-state skew
        red.reduce(g, out=out)
    torch.cuda.synchronize()
    if it >= 10:
        G = torch.cuda.get_device_properties(0).multi_processor_count * 8
        buf = (ctypes.c_uint64 * (8 * G))()
        check(lib.s2_p2p_trace(red.plan.handle, buf, 8 * G))
        t = np.frombuffer(buf, dtype=np.uint64).reshape(G, 8)[:, :5].astype(np.int64)
        t = t[t[:, 0] > 0]  # CTAs of the last launch
        for c in range(1, 5):  # slots a kernel does not stamp: carry the previous stamp
            miss = t[:, c] == 0
            t[miss, c] = t[miss, c - 1]
        t0 = t[:, 0].min()
        res.append({"ctas": int(len(t)), "start_spread": int(t[:, 0].max() - t0),
                    "s0_s1": int(np.median(t[:, 1] - t[:, 0])), "s1_s2": int(np.median(t[:, 2] - t[:, 1])),
                    "s2_s3": int(np.median(t[:, 3] - t[:, 2])), "s3_s4": int(np.median(t[:, 4] - t[:, 3])),
                    "total": int(t[:, 4].max() - t0)})
agg = {k: int(np.median([r[k] for r in res])) for k in res[0]}
all_ = [None] * world
dist.all_gather_object(all_, agg)
if rank == 0:
    print(json.dumps({"ns_median": all_}))
dist.destroy_process_group()
