"""DDP (world 1, NCCL) with the S2 comm hook and error feedback, several gradient buckets.

Run by tests/test_training_loop.py in a subprocess (process-global torch.distributed state).
Per step and bucket it checks, with e = the hook's residual before the call and raw = the
bucket gradient DDP handed in:
  * the estimate DDP receives equals the oracle decode of g~ = raw + e (casq.py:329-331)
    within the fp32 tolerance (1e-5 x cell L1 mass);
  * the carried residual is exactly g~ - estimate (casq.py:331);
  * residuals follow the bucket's PARAMETERS across DDP's bucket rebuild (no shape errors,
    no residual of another bucket added), and stale residuals are dropped.
Prints one JSON line.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.nn as nn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import s2_oracle as o  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{os.environ.get('S2_TEST_PORT', '29611')}",
                        rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_2110_02140_b200.ddp import S2HookState, s2_comm_hook  # noqa: E402

torch.manual_seed(0)


class Model(nn.Module):
    def __init__(self):
        super().__init__()
        self.e1 = nn.Embedding(3000, 8)
        self.e2 = nn.Embedding(2000, 8)
        self.l1 = nn.Linear(16, 8)
        self.l2 = nn.Linear(8, 1)

    def forward(self, a, b):
        h = torch.cat([self.e1(a).mean(1), self.e2(b).mean(1)], -1)
        return self.l2(torch.relu(self.l1(h))).squeeze(-1)


model = Model().cuda()
ddp = nn.parallel.DistributedDataParallel(model, device_ids=[0], bucket_cap_mb=0.05)
state = S2HookState(size_ratio=4.0, alpha=0.2, seed=3, error_feedback=True)
LOG = []


def hook(st, bucket):
    key = tuple(id(p) for p in bucket.parameters())
    raw = bucket.buffer().clone().reshape(-1)
    prev = st.residuals.get(key)
    e_prev = prev.e.clone() if prev is not None and prev.e.numel() == raw.numel() else torch.zeros_like(raw)
    fut = s2_comm_hook(st, bucket)
    est = bucket.buffer().clone().reshape(-1)
    LOG.append((key, raw, e_prev, est, st.residuals[key].e.clone(), st.reducers[raw.numel()].cols))
    return fut


ddp.register_comm_hook(state, hook)
rng = torch.Generator(device="cuda")
rng.manual_seed(7)
report = {"steps": [], "ok": True}
for step in range(4):
    LOG.clear()
    a = torch.randint(0, 3000, (32, 4), device="cuda", generator=rng)
    b = torch.randint(0, 2000, (32, 4), device="cuda", generator=rng)
    loss = (ddp(a, b) ** 2).mean()
    ddp.zero_grad()
    loss.backward()
    torch.cuda.synchronize()
    srep = {"buckets": len(LOG), "max_err_over_tol": 0.0, "residual_exact": True, "outside_zero": True}
    for key, raw, e_prev, est, e_new, cols in LOG:
        g_t = (raw + e_prev)
        srep["residual_exact"] &= bool(torch.equal(e_new, g_t - est))
        gt = g_t.cpu().numpy().astype(np.float64)
        flags = gt != 0
        ref = o.decompress(o.compress(gt, flags, 3, cols, 3))
        idx = np.flatnonzero(flags)
        mass = o.sketch_l1_mass(o.row_seeds(3, 3), idx, gt[idx], cols)
        mmax = np.zeros(gt.size)
        for j, s in enumerate(o.row_seeds(3, 3)):
            mmax[idx] = np.maximum(mmax[idx], mass[j, o.hash_buckets(s, idx, cols)])
        err = np.abs(est.cpu().numpy().astype(np.float64) - ref)
        srep["max_err_over_tol"] = max(srep["max_err_over_tol"], float((err / np.maximum(1e-5 * mmax, 1e-30)).max()))
        srep["outside_zero"] &= bool(not est.cpu().numpy()[~flags].any())
    srep["residuals_held"] = len(state.residuals)
    srep["residual_nonzero"] = any(bool(x.e.abs().sum() > 0) for x in state.residuals.values())
    report["steps"].append(srep)
    report["ok"] &= (srep["residual_exact"] and srep["max_err_over_tol"] <= 1.0 and srep["outside_zero"]
                     and srep["residuals_held"] == srep["buckets"])
# DDP starts with one large first bucket and rebuilds into several after iteration 1: the
# residual of the old bucket must be dropped, not added to a differently shaped bucket
nb = [st["buckets"] for st in report["steps"]]
report["rebuilt"] = len(set(nb)) > 1
report["ok"] &= report["steps"][-1]["residual_nonzero"] and max(nb) >= 2 and report["rebuilt"]
state.check()
print(json.dumps(report), flush=True)
dist.destroy_process_group()
sys.exit(0 if report["ok"] else 1)
