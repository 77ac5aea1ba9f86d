"""The W > 1 exchange on ONE GPU: W virtual ranks (own plans, arenas and streams, no NCCL)
run the product's peer-memory exchange kernels (k_p2p_oneshot / k_p2p_aggregate), so a
single-GPU box checks W = 2..8 — including the north-star W = 8 — against the oracle's
sparse_merge + sparse_decompress (sparse.py:174-214).

Bar: integer inputs bit-exact; real-valued inputs within
1e-5 * max_j M[j, h_j(i)] / W; every rank's output bit-identical (replicated decode).
"""

import os

import numpy as np
import pytest

from oracle import s2_oracle as o

pytestmark = pytest.mark.gpu


def _reference(grads, nb, rows, cols, seed, kind):
    dim = grads[0].size
    ps = [o.compress(g, o.nonzero_flags(g, nb), rows, cols, seed) for g in grads]
    m = o.merge(ps)
    ref = o.decompress(m)
    mmax = None
    if kind != "int":
        mass = np.zeros((rows, cols))
        for g, p in zip(grads, ps):
            idx = o.selected_indices(p.flags, dim)
            idx = idx[g[idx] != 0]
            mass += o.sketch_l1_mass(o.row_seeds(seed, rows), idx, g[idx].astype(np.float64), cols)
        sel = o.selected_indices(m.flags, dim)
        mmax = np.zeros(dim)
        for j, s in enumerate(o.row_seeds(seed, rows)):
            mmax[sel] = np.maximum(mmax[sel], mass[j, o.hash_buckets(s, sel, cols)])
    return ref, m, mmax


def _check(outs, ref, mmax, W, kind):
    h0 = outs[0]
    for r, out in enumerate(outs):
        assert np.array_equal(out, h0), f"rank {r} differs from rank 0 (replicated decode)"
    if kind == "int":
        assert np.array_equal(h0, ref.astype(np.float32)), np.abs(h0 - ref).max()
    else:
        err = np.abs(h0.astype(np.float64) - ref)
        assert (err <= 1e-5 * mmax / W + 1e-30).all(), (err / np.maximum(mmax / W, 1e-30)).max()


CASES = [  # (W, one-shot max W, num_blocks divisor, rows, cols, push)
    (2, 2, 1, 3, 20011, 0),      # default one-shot
    (2, 1, 1, 3, 20011, 0),      # two-shot at W = 2
    (3, 2, 1, 3, 20011, 0),      # two-shot, W not a power of two (IEEE ÷3)
    (3, 4, 1, 5, 65536, 0),      # one-shot at W = 3
    (4, 2, 1, 3, 262144, 0),     # default two-shot
    (4, 4, 1, 3, 20011, 0),      # one-shot at W = 4
    (4, 2, 32, 3, 20011, 0),     # block bitmap, 32 elements per block
    (5, 2, 1, 3, 20011, 0),
    (6, 2, 1, 5, 1_000_000, 0),  # BERT-like non-power-of-two width
    (7, 2, 7, 3, 4099, 0),       # ragged blocks
    (8, 2, 1, 3, 262144, 0),     # the north-star W = 8
    (8, 2, 1, 3, 20011, 0),
    # push exchange (S2_P2P_PUSH=1): data stored into the peers' inboxes before each flag
    (2, 2, 1, 3, 20011, 1),
    (3, 4, 1, 5, 65536, 1),
    (4, 4, 32, 3, 20011, 1),
    (2, 1, 1, 3, 20011, 1),
    (4, 2, 1, 3, 262144, 1),
    (7, 2, 7, 3, 4099, 1),
    (8, 2, 1, 3, 262144, 1),
]


@pytest.mark.parametrize("W,oneshot_maxw,bdiv,rows,cols,push", CASES)
def test_local_exchange_parity(W, oneshot_maxw, bdiv, rows, cols, push):
    import torch

    from paper_2110_02140_b200.local import LocalGroup

    dim = 2_000_003
    nb = dim if bdiv == 1 else -(-dim // bdiv)
    env = {"S2_P2P_ONESHOT_MAXW": str(oneshot_maxw), "S2_P2P_PUSH": str(push)}  # read at arena layout
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        grp = LocalGroup(W, dim, rows, cols, seed=0, num_blocks=nb)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
    words = torch.zeros(W, dtype=torch.int32, device="cuda")
    grp.set_status(words)
    # three inputs with different non-zero positions, each reduced twice (six reduces cover every
    # table slot of the period-4 rotation): a stale bitmap or table would fail parity
    for kind, base in (("int", 1234), ("normal", 1234), ("normal", 4321)):
        grads = [o.synthetic_gradient(dim, 0.01, r, kind=kind, base_seed=base) for r in range(W)]
        ref, _, mmax = _reference(grads, nb, rows, cols, 0, kind)
        gt = [torch.from_numpy(g).cuda() for g in grads]
        for _ in range(2):
            outs = grp.reduce(gt)
            torch.cuda.synchronize()
            _check([x.cpu().numpy() for x in outs], ref, mmax, W, kind)
            assert words.cpu().tolist() == [0] * W
    assert grp.errors() == [0] * W


def test_local_exchange_timeout_poisons_output():
    """A rank that never arrives: the waiting rank's barrier gives up after the timeout, the
    output is all NaN (never a silently incomplete average) and the status word says so;
    later reduces stay NaN without waiting again (the error is sticky)."""
    import time

    import torch

    from paper_2110_02140_b200._lib import S2_STATUS_EXCHANGE, check, lib, ptr
    from paper_2110_02140_b200.local import LocalGroup

    dim = 100_000
    grp = LocalGroup(2, dim, 3, 1667, timeout_s=0.5)
    words = torch.zeros(2, dtype=torch.int32, device="cuda")
    grp.set_status(words)
    g = torch.from_numpy(o.synthetic_gradient(dim, 0.01, 0, kind="int")).cuda()
    out = torch.zeros(dim, device="cuda")
    import ctypes

    t0 = time.time()
    check(lib.s2_reduce(grp.plans[0].handle, ptr(g), ptr(out), None, ctypes.c_void_p(0)))  # rank 1 never comes
    torch.cuda.synchronize()
    assert time.time() - t0 < 30
    assert torch.isnan(out).all()
    assert int(words[0]) == S2_STATUS_EXCHANGE
    assert lib.s2_p2p_error(grp.plans[0].handle) != 0
    t0 = time.time()
    out.zero_()
    check(lib.s2_reduce(grp.plans[0].handle, ptr(g), ptr(out), None, ctypes.c_void_p(0)))
    torch.cuda.synchronize()
    assert time.time() - t0 < 0.4, "a plan that timed out must not wait again"
    assert torch.isnan(out).all()


def test_reducer_async_status_raises_on_next_call():
    """S2Reducer surfaces the previous step's NaN/Inf flag on a later call without syncing."""
    import torch

    import paper_2110_02140_b200 as s2

    d = 100_000
    red = s2.S2Reducer(d, rows=3, cols=1667)
    g = torch.from_numpy(o.synthetic_gradient(d, 0.01, 0, kind="int")).cuda()
    red.reduce(g)
    red.check()
    bad = g.clone()
    bad[5] = float("nan")
    red.reduce(bad)
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="gradient vector contains NaN or Inf"):
        red.reduce(g)
    red.reduce(g)
    red.check()  # healthy again


@pytest.mark.parametrize("W,push", [(2, 0), (4, 1), (8, 1)])
def test_local_back_to_back(W, push):
    """Eight W-rank reduces launched back to back with no host sync (every buffer slot of the
    rotation in flight, compress i+1 overlapping decode i), all outputs checked afterwards."""
    import torch

    from paper_2110_02140_b200.local import LocalGroup

    dim, rows, cols = 500_009, 3, 4099
    old = os.environ.get("S2_P2P_PUSH")
    os.environ["S2_P2P_PUSH"] = str(push)
    try:
        grp = LocalGroup(W, dim, rows, cols)
    finally:
        if old is None:
            os.environ.pop("S2_P2P_PUSH")
        else:
            os.environ["S2_P2P_PUSH"] = old
    steps = []
    for k in range(8):
        grads = [o.synthetic_gradient(dim, 0.01 * (1 + k % 3), r, kind="int", base_seed=100 * k) for r in range(W)]
        outs = grp.reduce([torch.from_numpy(g).cuda() for g in grads])
        steps.append((grads, outs))
    torch.cuda.synchronize()
    for k, (grads, outs) in enumerate(steps):
        ref = o.decompress(o.merge([o.compress(g, g != 0, rows, cols, 0) for g in grads])).astype(np.float32)
        for r, out in enumerate(outs):
            assert np.array_equal(out.cpu().numpy(), ref), (k, r)
    assert grp.errors() == [0] * W


@pytest.mark.parametrize("W,push,oneshot_maxw", [(2, 0, 2), (2, 1, 1), (4, 1, 2), (4, 0, 2), (8, 1, 2)])
def test_local_reduce_many_pipelined(W, push, oneshot_maxw):
    """s2_reduce_many with W > 1 pipelines the batch (compress k+1 beside exchange k, then decode k);
    six steps of different inputs, every rank's output of every step against the oracle."""
    import torch

    from paper_2110_02140_b200.local import LocalGroup

    dim, rows, cols = 400_009, 3, 4099
    env = {"S2_P2P_PUSH": str(push), "S2_P2P_ONESHOT_MAXW": str(oneshot_maxw)}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        grp = LocalGroup(W, dim, rows, cols)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
    words = torch.zeros(W, dtype=torch.int32, device="cuda")
    grp.set_status(words)
    host = [[o.synthetic_gradient(dim, 0.005 * (1 + k % 4), r, kind="int", base_seed=77 * k) for r in range(W)]
            for k in range(6)]
    outs = grp.reduce_many([[torch.from_numpy(g).cuda() for g in step] for step in host])
    torch.cuda.synchronize()
    for k, step in enumerate(host):
        ref = o.decompress(o.merge([o.compress(g, g != 0, rows, cols, 0) for g in step])).astype(np.float32)
        for r in range(W):
            assert np.array_equal(outs[k][r].cpu().numpy(), ref), (k, r)
    assert words.cpu().tolist() == [0] * W and grp.errors() == [0] * W


@pytest.mark.parametrize("W,push", [(2, 0), (4, 1)])
def test_local_exchange_beside_concurrent_compute(W, push):
    """The exchange kernels spin on cross-rank flags while other streams keep the SMs busy (the
    DDP situation: the comm hook's stream overlaps backward kernels).  A side stream runs large
    matmuls launched before and between the reduces; every reduce must still complete — no
    barrier timeout — and match the oracle bit for bit."""
    import torch

    from paper_2110_02140_b200.local import LocalGroup

    dim, rows, cols = 1_000_003, 3, 20011
    old = os.environ.get("S2_P2P_PUSH")
    os.environ["S2_P2P_PUSH"] = str(push)
    try:
        grp = LocalGroup(W, dim, rows, cols, timeout_s=20.0)
    finally:
        if old is None:
            os.environ.pop("S2_P2P_PUSH")
        else:
            os.environ["S2_P2P_PUSH"] = old
    words = torch.zeros(W, dtype=torch.int32, device="cuda")
    grp.set_status(words)
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda")
    b = torch.randn(4096, 4096, device="cuda")
    cs = []
    steps = []
    for k in range(4):
        with torch.cuda.stream(side):
            for _ in range(4):
                cs.append(a @ b)  # occupies every SM for tens of microseconds per launch
        grads = [o.synthetic_gradient(dim, 0.01, r, kind="int", base_seed=31 * k + 5) for r in range(W)]
        outs = grp.reduce([torch.from_numpy(g).cuda() for g in grads])
        steps.append((grads, outs))
    torch.cuda.synchronize()
    for k, (grads, outs) in enumerate(steps):
        ref = o.decompress(o.merge([o.compress(g, g != 0, rows, cols, 0) for g in grads])).astype(np.float32)
        for r, out in enumerate(outs):
            assert np.array_equal(out.cpu().numpy(), ref), (k, r)
    assert words.cpu().tolist() == [0] * W and grp.errors() == [0] * W
    assert torch.isfinite(cs[-1]).all()


@pytest.mark.parametrize("W,n", [(2, 1), (2, 2), (4, 2), (4, 3)])
def test_local_reduce_many_short_batches(W, n):
    """Batches of 1..3 reduces (the two-stream schedule's first compress waits up front; n = 1 stays
    on one stream), back to back with single reduces on the same plans, all checked."""
    import torch

    from paper_2110_02140_b200.local import LocalGroup

    dim, rows, cols = 300_007, 3, 4099
    grp = LocalGroup(W, dim, rows, cols)
    host = [[o.synthetic_gradient(dim, 0.01 * (1 + k), r, kind="int", base_seed=13 * k + 1) for r in range(W)]
            for k in range(n + 1)]
    outs = grp.reduce_many([[torch.from_numpy(g).cuda() for g in step] for step in host[:n]])
    single = grp.reduce([torch.from_numpy(g).cuda() for g in host[n]])  # a plain reduce right after the batch
    again = grp.reduce_many([[torch.from_numpy(g).cuda() for g in step] for step in host[:n]])
    torch.cuda.synchronize()
    for k, step in enumerate(host):
        ref = o.decompress(o.merge([o.compress(g, g != 0, rows, cols, 0) for g in step])).astype(np.float32)
        got = [single] if k == n else [outs[k], again[k]]
        for res in got:
            for r in range(W):
                assert np.array_equal(res[r].cpu().numpy(), ref), (k, r)
    assert grp.errors() == [0] * W


@pytest.mark.parametrize("W", [2, 4])
def test_local_reduce_many_block_bitmap(W):
    """Pipelined batches with a block bitmap (b < d, ragged last block): the block decode keeps a
    zeroed value stage across tiles and reduces of the batch; every output against the oracle."""
    import torch

    from paper_2110_02140_b200.local import LocalGroup

    dim, rows, cols, bs = 250_007, 3, 4099, 40
    nb = -(-dim // bs)
    grp = LocalGroup(W, dim, rows, cols, num_blocks=nb)
    host = []
    for k in range(5):
        step = []
        for r in range(W):
            rng = np.random.default_rng(1000 * k + r)
            g = np.zeros(dim, np.float32)
            for b in rng.choice(nb, max(1, nb // (50 * (1 + k % 2))), replace=False):
                lo, hi = b * bs, min(dim, (b + 1) * bs)
                g[lo:hi] = rng.integers(-1000, 1000, hi - lo).astype(np.float32)
            step.append(g)
        host.append(step)
    outs = grp.reduce_many([[torch.from_numpy(g).cuda() for g in step] for step in host])
    torch.cuda.synchronize()
    for k, step in enumerate(host):
        ps = [o.compress(g, o.nonzero_flags(g, nb), rows, cols, 0) for g in step]
        ref = o.decompress(o.merge(ps)).astype(np.float32)
        for r in range(W):
            assert np.array_equal(outs[k][r].cpu().numpy(), ref), (k, r)
    assert grp.errors() == [0] * W
