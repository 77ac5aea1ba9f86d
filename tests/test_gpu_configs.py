"""GPU parity at the BASELINE.json configs beyond the 1M/25.6M cases (W = 1):
BERT-base 110M / 95% / 5 x 1,000,000 (non-power-of-two magic-divide path), LSTM embedding
200M / 99.9% row-sparse with element and row (b = 200k) bitmaps, GPT-2-M 355M / 90% (bitmap,
nnz and sketch row-sum properties, then the full table and a 1M-coordinate decode sample against
a float64 reference), BERT 5 x 2^20 likewise.  Tolerance as in test_gpu_parity (L1-mass relative)."""
import numpy as np
import pytest

from oracle import s2_oracle as o

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _cuda(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _check(g, nb, rows, cols, seed=0):
    import paper_2110_02140_b200 as s2

    p = s2.sparse_compress(_cuda(g), None, rows, cols, seed, num_blocks=nb)
    flags = o.nonzero_flags(g, nb)
    assert np.array_equal(p.mask.words.cpu().numpy().view(np.uint32), o.mask_words(flags))
    ref = o.compress(g, flags, rows, cols, seed)
    idx = o.selected_indices(flags, g.size)
    v = g.astype(np.float64)[idx]
    nz = v != 0
    mass = o.sketch_l1_mass(o.row_seeds(seed, rows), idx[nz], v[nz], cols)
    tab = p.table.table.cpu().numpy().astype(np.float64)
    assert (np.abs(tab - ref.table) <= TOL * mass + 1e-30).all()
    out = s2.sparse_decompress(p).cpu().numpy()
    ref_out = o.decompress(ref)
    mmax = np.zeros(idx.size)
    for j, s in enumerate(o.row_seeds(seed, rows)):
        mmax = np.maximum(mmax, mass[j, o.hash_buckets(s, idx, cols)])
    assert (np.abs(out[idx].astype(np.float64) - ref_out[idx]) <= TOL * mmax + 1e-30).all()
    outside = np.ones(g.size, bool)
    outside[idx] = False
    assert not out[outside].any()


def _rows_gradient(V, H, frac, rank=0):
    rng = np.random.default_rng(1234 + rank)
    g = np.zeros(V * H, np.float32)
    for r in rng.choice(V, max(1, int(round(frac * V))), replace=False):
        g[r * H:(r + 1) * H] = rng.standard_normal(H).astype(np.float32)
    return g


def test_bert_110m_5x1000000():
    d = 110_000_000
    _check(o.synthetic_gradient(d, 0.05, 0), d, 5, 1_000_000)


def test_lstm_200m_rows_element_and_row_bitmaps():
    V, H = 200_000, 1_000
    g = _rows_gradient(V, H, 0.001)
    _check(g, V * H, 3, 1_048_576)  # element bitmap
    _check(g, V, 3, 1_048_576)      # one bit per embedding row


def _check_full_size(g, rows, cols, seed=0, sample=1_000_000):
    """Full-size W = 1 parity for a CUDA gradient too large for the np.add.at oracle path:
    bitmap bit-exact (packed on the GPU), nnz exact, the whole table against a float64 reference
    table built per row with np.bincount over the oracle's hashes (core.py:70-106), and the decode
    on `sample` random union coordinates against the float64 lower-median query of that table
    (sketch.py:114-128); zeros outside the union checked on the GPU."""
    import torch

    import paper_2110_02140_b200 as s2

    d = g.numel()
    p = s2.sparse_compress(g, None, rows, cols, seed)
    nzmask = g != 0
    pad = (-d) % 32
    bits = torch.cat([nzmask, torch.zeros(pad, dtype=torch.bool, device=g.device)]).view(-1, 32).to(torch.int64)
    ref_words = (bits << torch.arange(32, device=g.device)).sum(1)
    assert torch.equal(p.mask.words.to(torch.int64) & 0xFFFFFFFF, ref_words & 0xFFFFFFFF)
    del bits, ref_words
    assert p.nnz == int(nzmask.sum())
    idx = torch.nonzero(nzmask).reshape(-1).cpu().numpy()
    vals = g[nzmask].double().cpu().numpy()
    tab = p.table.table.double().cpu().numpy()
    seeds = o.row_seeds(seed, rows)
    ref = np.zeros((rows, cols))
    mass = np.zeros((rows, cols))
    for j, s in enumerate(seeds):
        b = o.hash_buckets(s, idx, cols)
        ref[j] = np.bincount(b, weights=o.hash_signs(s, idx) * vals, minlength=cols)
        mass[j] = np.bincount(b, weights=np.abs(vals), minlength=cols)
    assert (np.abs(tab - ref) <= TOL * mass + 1e-30).all(), float((np.abs(tab - ref) / np.maximum(mass, 1e-30)).max())
    out = s2.sparse_decompress(p)
    assert not bool(out[~nzmask].any()), "non-zero outside the union bitmap"
    rng = np.random.default_rng(99)
    smp = np.sort(rng.choice(idx, min(sample, idx.size), replace=False))
    got = out[torch.from_numpy(smp).cuda()].double().cpu().numpy()
    est = np.stack([o.hash_signs(s, smp) * ref[j, o.hash_buckets(s, smp, cols)] for j, s in enumerate(seeds)])
    est.sort(axis=0)
    want = est[(rows - 1) // 2]
    mmax = np.zeros(smp.size)
    for j, s in enumerate(seeds):
        mmax = np.maximum(mmax, mass[j, o.hash_buckets(s, smp, cols)])
    assert (np.abs(got - want) <= TOL * mmax + 1e-30).all()


def test_gpt2m_355m_90pct_full_parity():
    """GPT-2-M 355M / 90 % / 3 x 2^20 (BASELINE configs[4], densest sweep point) at W = 1."""
    from paper_2110_02140_b200 import synthetic

    _check_full_size(synthetic.cuda_gradient(355_000_000, 0.10, 0), 3, 1_048_576)


def test_bert_110m_5x2pow20_full_parity():
    """BERT-base 110M / 95 % / 5 x 2^20 — the bench.py `bert` config — at W = 1."""
    from paper_2110_02140_b200 import synthetic

    _check_full_size(synthetic.cuda_gradient(110_000_000, 0.05, 0), 5, 1_048_576)


def test_gpt2m_355m_90pct_properties():
    """Full-size properties: bitmap bit-exact, nnz exact, and per sketch row the sum of cells
    equals sum_i s_j(i) v_i (linearity) within the L1 bound."""
    import torch

    import paper_2110_02140_b200 as s2
    from paper_2110_02140_b200 import synthetic

    d, rows, cols = 355_000_000, 3, 1_048_576
    g = synthetic.cuda_gradient(d, 0.10, 0)
    p = s2.sparse_compress(g, None, rows, cols, 0)
    nzmask = g != 0
    words = p.mask.words
    # bitmap from torch: pack g != 0 little-endian into int32 words on the GPU
    pad = (-d) % 32
    bits = torch.cat([nzmask, torch.zeros(pad, dtype=torch.bool, device=g.device)]).view(-1, 32).to(torch.int64)
    ref_words = (bits << torch.arange(32, device=g.device)).sum(1).to(torch.int64)
    assert torch.equal(words.to(torch.int64) & 0xFFFFFFFF, ref_words & 0xFFFFFFFF)
    assert p.nnz == int(nzmask.sum())
    idx = torch.nonzero(nzmask).reshape(-1).cpu().numpy()
    vals = g[nzmask].double().cpu().numpy()
    tab = p.table.table.double().cpu().numpy()
    for j, s in enumerate(o.row_seeds(0, rows)):
        sg = o.hash_signs(s, idx)
        want = float((sg * vals).sum())
        assert abs(tab[j].sum() - want) <= TOL * float(np.abs(vals).sum())
