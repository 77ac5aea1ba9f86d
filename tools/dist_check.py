"""Multi-GPU parity of S2Reducer (one process per GPU, NCCL over NVLink) against the oracle.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P tools/dist_check.py [--dim D]

Every rank reduces its own synthetic gradient (seed 1234 + rank); every rank
re-derives all W gradients on the host and checks its output against
oracle.decompress(oracle.merge(oracle.compress(g_r) for r)):
  * integer-valued inputs: bit-exact;
  * real-valued inputs: within 1e-5 x the cell L1 mass;
and all ranks must hold identical outputs (replicated decode).  Prints one JSON line.
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import s2_oracle as o  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=2_000_000)
ap.add_argument("--alpha", type=float, default=0.01)
ap.add_argument("--cols", type=int, default=20011)
ap.add_argument("--rows", type=int, default=3)
a = ap.parse_args()

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
import paper_2110_02140_b200 as s2  # noqa: E402

nb = int(os.environ.get("S2_CHECK_NUM_BLOCKS", "0")) or a.dim  # block bitmap (b < d) when set
red = s2.S2Reducer(a.dim, rows=a.rows, cols=a.cols, seed=0, num_blocks=nb)
graphed = None
if os.environ.get("S2_CHECK_GRAPH") == "1":  # replay captured CUDA graphs instead of direct calls
    from paper_2110_02140_b200.reducer import GraphedReduce

    g_static = torch.zeros(a.dim, device="cuda")
    out_static = torch.empty(a.dim, device="cuda")
    graphed = GraphedReduce(red, g_static, out_static)
report = {"world": world, "dim": a.dim, "graph": graphed is not None}
# three inputs with different non-zero positions (base seeds), each reduced twice, every
# output checked: a stale bitmap or table from the previous call of the same ping-pong
# parity would show up as a parity failure
CASES = (("int", "int", 1234), ("normal", "normal", 1234), ("normal_b", "normal", 4321))
MANY = os.environ.get("S2_CHECK_MANY") == "1"  # the pipelined batch API (reduce_many) instead


def expected(kind, base):
    grads = [o.synthetic_gradient(a.dim, a.alpha, r, kind=kind, base_seed=base) for r in range(world)]
    ps = [o.compress(g, o.nonzero_flags(g, nb), a.rows, a.cols, 0) for g in grads]
    m = o.merge(ps)
    ref = o.decompress(m)
    union = o.selected_indices(m.flags, a.dim)
    mmax = None
    if kind != "int":
        mass = np.zeros((a.rows, a.cols))
        for g, p in zip(grads, ps):
            idx = o.selected_indices(p.flags, a.dim)
            idx = idx[g[idx] != 0]
            mass += o.sketch_l1_mass(o.row_seeds(0, a.rows), idx, g[idx].astype(np.float64), a.cols)
        mmax = np.zeros(union.size)
        for j, s in enumerate(o.row_seeds(0, a.rows)):
            mmax = np.maximum(mmax, mass[j, o.hash_buckets(s, union, a.cols)])
    outside = np.ones(a.dim, bool)
    outside[union] = False
    return grads[rank], ref, union, mmax, outside, int(m.flags.sum())


exp = {name: expected(kind, base) for name, kind, base in CASES}
many_outs = {}
if MANY:  # one pipelined batch cycling through the three inputs twice, every output checked
    seq = [c[0] for c in CASES] * 2
    batch = red.reduce_many([torch.from_numpy(exp[n][0]).cuda() for n in seq])
    for n, x in zip(seq, batch):
        many_outs.setdefault(n, []).append(x.cpu().numpy())
for name, kind, base in CASES:
    g_rank, ref, union, mmax, outside, nnz_union = exp[name]
    oks_rep, errs, hashes = [], [], []
    outs_many = many_outs.get(name, [])
    for rep in range(len(outs_many) if MANY else 2):  # every buffer slot of the rotation
        if MANY:
            out = outs_many[rep]
        elif graphed is None:
            out = red.reduce(torch.from_numpy(g_rank).cuda()).cpu().numpy()
        else:
            g_static.copy_(torch.from_numpy(g_rank))
            out = graphed().cpu().numpy()
        if kind == "int":
            oks_rep.append(bool(np.array_equal(out, ref.astype(np.float32))))
            errs.append(float(np.abs(out - ref).max()))
        else:
            e = np.abs(out[union].astype(np.float64) - ref[union])
            oks_rep.append(bool((e <= 1e-5 * mmax / world + 1e-30).all() and not out[outside].any()))
            errs.append(float((e / np.maximum(mmax / world, 1e-30)).max()))
        hashes.append(hashlib.sha256(out.tobytes()).hexdigest())
    hs = [None] * world
    dist.all_gather_object(hs, hashes)
    report[name] = {"parity": all(oks_rep) and len(oks_rep) > 0, "max_err": max(errs),
                    "replicated": all(len({h[k] for h in hs}) == 1 for k in range(len(hashes))),
                    "nnz_union": nnz_union}
oks = [None] * world
dist.all_gather_object(oks, all(report[c[0]]["parity"] and report[c[0]]["replicated"] for c in CASES))
report["all_ranks_ok"] = all(oks)
if rank == 0:
    print(json.dumps(report), flush=True)
dist.destroy_process_group()
sys.exit(0 if report["all_ranks_ok"] else 1)
