"""GPU parity of the sm_100a S2 path against the golden vectors and the CPU oracle.

Bar:
  * bitmaps, compacted indices, union bitmaps: bit-exact;
  * integer-valued inputs: sketch tables and decoded gradients bit-exact
    (== float32 of the float64 reference) — every partial sum is an integer < 2^24;
  * real-valued inputs: |T_gpu - T_ref| <= TOL * M per cell, M = sum of |v| over the
    cell's contributions (the fp32 summation-order bound); decode within
    TOL * max_j M[j, h_j(i)] / W (the lower median is 1-Lipschitz in max-norm).
"""

import glob
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import s2_oracle as o

pytestmark = pytest.mark.gpu
TOL = 1e-5  # relative to the cell's L1 mass (north_star: <= 1e-5, summation order only)

CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "s2_*.npz")))


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="module")
def s2():
    import torch

    assert torch.cuda.is_available()
    import paper_2110_02140_b200 as s2mod

    return s2mod


def cuda(x):
    import torch

    return torch.as_tensor(np.ascontiguousarray(x)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def words_u32(t):
    return host(t).astype(np.int32).view(np.uint32)


def cell_mass(g, flags, rows, cols, seed):
    idx = o.selected_indices(flags, g.size)
    v = g.astype(np.float64)[idx]
    nz = v != 0
    return o.sketch_l1_mass(o.row_seeds(seed, rows), idx[nz], v[nz], cols)


def assert_table_close(got, ref, mass, exact):
    if exact:
        assert np.array_equal(got, ref.astype(np.float32)), np.abs(got - ref).max()
    else:
        err = np.abs(got.astype(np.float64) - ref)
        assert (err <= TOL * mass + 1e-30).all(), (err / np.maximum(mass, 1e-30)).max()


def assert_decode_close(got, ref_out, union_idx, mass, seeds, cols, W, exact):
    dim = got.size
    outside = np.ones(dim, bool)
    outside[union_idx] = False
    assert not got[outside].any(), "non-zero outside the union bitmap"
    g_u = got[union_idx].astype(np.float64)
    r_u = ref_out
    if exact:
        assert np.array_equal(got[union_idx], r_u.astype(np.float32))
        return
    mmax = np.zeros(union_idx.size)
    for j, s in enumerate(seeds):
        mmax = np.maximum(mmax, mass[j, o.hash_buckets(s, union_idx, cols)])
    err = np.abs(g_u - r_u)
    assert (err <= TOL * mmax / W + 1e-30).all(), (err / np.maximum(mmax / W, 1e-30)).max()


@pytest.mark.parametrize("name", CASES)
def test_golden_case(s2, name):
    """Every worker's compress, the merge and the decode against the live-reference fixture."""
    z = load(name)
    dim, nb, rows, cols, seed, W = (int(z[k]) for k in ("dim", "num_blocks", "rows", "cols", "seed", "W"))
    # integer-valued inputs, also in units of 2^-149 (fp32 subnormals): every sum is exact
    exact = name in ("s2_int_w8", "s2_r4", "s2_subnormal_int")
    part = s2.BlockPartition(dim, nb)
    payloads = []
    for w in range(W):
        g = z["grads"][w]
        if name == "s2_blocks_topk":
            mask = s2.BlockMask(part, o.words_to_flags(z["words"][w], nb))
            p = s2.sparse_compress(cuda(g), mask, rows, cols, seed)
        else:
            p = s2.sparse_compress(cuda(g), None, rows, cols, seed, num_blocks=nb)
        assert np.array_equal(words_u32(p.mask.words), z["words"][w])
        assert p.alpha == z["alphas"][w]
        flags = o.words_to_flags(z["words"][w], nb)
        assert_table_close(host(p.table.table), z["tables"][w], cell_mass(g, flags, rows, cols, seed), exact)
        payloads.append(p)
    if exact:
        wire = payloads[0].to_bytes()
        assert hashlib.sha256(wire).digest() == z["wire_sha256"].tobytes()
    assert np.array_equal(np.frombuffer(payloads[0].to_bytes()[:53], np.uint8), z["wire_head"])
    assert payloads[0].serialized_nbytes() == int(z["nbytes"])
    c = s2.sparse_comm_bits(payloads[0])  # CommCost, sparse.py:244-285
    assert [c.payload_bits, c.dense_bits, c.coordinate_bits, c.value_bits, c.bitmap_bits,
            c.header_bits] == z["comm_bits"].tolist()
    m = s2.sparse_merge(payloads)
    assert m.workers == W
    cm = s2.sparse_comm_bits(m)
    assert [cm.payload_bits, cm.dense_bits, cm.coordinate_bits, cm.value_bits, cm.bitmap_bits,
            cm.header_bits] == z["comm_bits_merged"].tolist()
    assert cm.ratio_vs_dense == cm.payload_bits / cm.dense_bits
    assert np.array_equal(words_u32(m.mask.words), z["union_words"])
    assert m.alpha == float(z["merged_alpha"])
    assert_table_close(host(m.table.table), z["merged_table"], z["l1_mass"], exact)
    out = host(s2.sparse_decompress(m))
    assert np.array_equal(host(m.mask.selected_indices()), z["union_idx"])
    assert_decode_close(out, z["decode_at_union"], z["union_idx"], z["l1_mass"], o.row_seeds(seed, rows), cols, W,
                        exact)


def test_tiny_table_kat(s2):
    z = load("tiny_table")
    t = s2.CountSketchTable(3, 8, seed=0, dim=16)
    t.insert([1, 5, 9], [1.0, -2.0, 0.5])
    assert np.array_equal(host(t.table), z["table"].astype(np.float32))
    assert host(t.query([1, 5, 9])).tolist() == [1.0, -2.0, 0.5]


def test_device_hash_exact_via_integer_table(s2):
    """Distinct small integers at random indices: the fp32 table is exact, so equality with the
    oracle table (built from golden-pinned hashes) proves every device bucket and sign."""
    rng = np.random.default_rng(3)
    for cols in (16384, 1667, 262144, 1_000_000, 97, 2**20 + 7):
        dim = 5_000_000
        idx = np.sort(rng.choice(dim, 4000, replace=False))
        g = np.zeros(dim, np.float32)
        g[idx] = np.arange(1, 4001, dtype=np.float32)
        p = s2.sparse_compress(cuda(g), None, 5, cols, 12345)
        ref = o.compress(g, g != 0, 5, cols, 12345).table
        assert np.array_equal(host(p.table.table), ref.astype(np.float32)), cols


def test_full_size_resnet_config(s2):
    """configs[1] (25.6M, 99%, 3x262144) at W=1 against the fast oracle: bitmap bit-exact,
    compacted indices/values exact, table and decode within the L1-mass tolerance."""
    import torch

    d, alpha, rows, cols = 25_600_000, 0.01, 3, 262144
    g = o.synthetic_gradient(d, alpha, 0)
    gt = cuda(g)
    p = s2.sparse_compress(gt, None, rows, cols, 0)
    flags = g != 0
    assert np.array_equal(words_u32(p.mask.words), o.mask_words(flags))
    assert p.nnz == int(flags.sum())
    idx, vals = s2.compacted_values(gt, p.mask)
    ref_idx = np.flatnonzero(flags)
    assert np.array_equal(host(idx), ref_idx)
    assert np.array_equal(host(vals), g[ref_idx])
    refp = o.compress(g, flags, rows, cols, 0)
    mass = cell_mass(g, flags, rows, cols, 0)
    assert_table_close(host(p.table.table), refp.table, mass, False)
    out = host(s2.sparse_decompress(p))
    ref_out = o.decompress(refp)
    assert_decode_close(out, ref_out[ref_idx], ref_idx, mass, o.row_seeds(0, rows), cols, 1, False)
    torch.cuda.synchronize()


def test_reducer_single_gpu_equals_compress_decode(s2):
    import torch

    d = 1_000_000
    red = s2.S2Reducer(d, rows=3, cols=16384, seed=0)
    # consecutive reduces rotate the plan's tables over 4 slots (decode i zeroes slot i+2)
    for k, alpha in enumerate((0.01, 0.05, 0.001, 0.02, 0.0, 0.03, 0.01, 0.2, 0.005)):
        g = o.synthetic_gradient(d, alpha, k, kind="int")
        out = host(red.reduce(cuda(g)))
        ref = o.decompress(o.compress(g, g != 0, 3, 16384, 0))
        assert np.array_equal(out, ref.astype(np.float32)), k
        assert red.last_nnz() == int((g != 0).sum())
    red.check_finite()
    bad = g.copy()
    bad[17] = np.inf
    red.reduce(cuda(bad))
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="NaN or Inf"):
        red.check_finite()


def test_nonfinite_and_errors(s2):
    g = np.zeros(1000, np.float32)
    g[3] = np.nan
    with pytest.raises(ValueError, match="gradient vector contains NaN or Inf"):
        s2.sparse_compress(cuda(g), None, 3, 16, 0)
    part = s2.BlockPartition(10, 10)
    with pytest.raises(ValueError, match="dimension mismatch: mask dim 10, vector 11"):
        s2.sparse_compress(cuda(np.ones(11, np.float32)), s2.BlockMask(part, np.ones(10, bool)), 3, 4, 0)
    p = s2.sparse_compress(cuda(np.ones(10, np.float32)), None, 3, 4, 0)
    with pytest.raises(ValueError, match="workers must be >= 1"):
        s2.sparse_decompress(p, workers=0)
    with pytest.raises(ValueError, match="nothing to merge"):
        s2.sparse_merge([])
    q = s2.sparse_compress(cuda(np.ones(10, np.float32)), None, 3, 5, 0)
    with pytest.raises(ValueError, match="incompatible payloads: field 'sketch_params' differs"):
        s2.sparse_merge([p, q])


def test_edge_shapes(s2):
    """ragged tails (d % 4, d % 32, d % 1024 != 0), d = 1, all-zero and all-dense vectors."""
    rng = np.random.default_rng(11)
    for d in (1, 2, 3, 5, 31, 33, 127, 1023, 1025, 4097, 100_003):
        for dens in (0.0, 0.3, 1.0):
            g = ((rng.random(d) < dens) * rng.integers(-50, 50, d)).astype(np.float32)
            p = s2.sparse_compress(cuda(g), None, 3, 7, 5)
            flags = g != 0
            assert np.array_equal(words_u32(p.mask.words), o.mask_words(flags)), (d, dens)
            ref = o.compress(g, flags, 3, 7, 5)
            assert np.array_equal(host(p.table.table), ref.table.astype(np.float32))
            out = host(s2.sparse_decompress(p))
            assert np.array_equal(out, o.decompress(ref).astype(np.float32)), (d, dens)


def test_block_masks(s2):
    """b < d: non-zero rule and given masks, ragged/empty tail blocks; decode fills whole blocks."""
    rng = np.random.default_rng(12)
    for d, nb in ((10_007, 1000), (5000, 7), (4099, 4098), (65_536, 2048), (1000, 1)):
        g = ((rng.random(d) < 0.01) * rng.integers(-9, 9, d)).astype(np.float32)
        p = s2.sparse_compress(cuda(g), None, 3, 64, 1, num_blocks=nb)
        flags = o.nonzero_flags(g, nb)
        assert np.array_equal(words_u32(p.mask.words), o.mask_words(flags)), (d, nb)
        assert p.alpha == o.selected_fraction(flags, d)
        ref = o.compress(g, flags, 3, 64, 1)
        assert np.array_equal(host(p.table.table), ref.table.astype(np.float32))
        assert np.array_equal(host(s2.sparse_decompress(p)), o.decompress(ref).astype(np.float32))
        assert np.array_equal(host(p.mask.selected_indices()), o.selected_indices(flags, d))
        # a given (random) mask: only non-zeros inside set blocks are inserted
        gflags = rng.random(nb) < 0.5
        q = s2.sparse_compress(cuda(g), s2.BlockMask(s2.BlockPartition(d, nb), gflags), 3, 64, 1)
        refq = o.compress(g, gflags, 3, 64, 1)
        assert np.array_equal(host(q.table.table), refq.table.astype(np.float32))
        assert q.alpha == o.selected_fraction(gflags, d)
        assert np.array_equal(host(s2.sparse_decompress(q)), o.decompress(refq).astype(np.float32))
        idx, vals = s2.compacted_values(cuda(g), q.mask)
        sel = o.selected_indices(gflags, d)
        nz = sel[g[sel] != 0]
        assert np.array_equal(host(idx), nz) and np.array_equal(host(vals), g[nz])


def test_mergeability_integer(s2):
    """Acceptance #7: merge-then-decompress == decompress of compress(sum) on the
    union mask, bit-exact on integer vectors, W in {2,4,8}."""
    d, rows, cols = 300_000, 3, 4099
    for W in (2, 4, 8):
        gs = [o.synthetic_gradient(d, 0.01, r, kind="int") for r in range(W)]
        m = s2.sparse_merge([s2.sparse_compress(cuda(g), None, rows, cols, 9) for g in gs])
        union = np.zeros(d, bool)
        for g in gs:
            union |= g != 0
        gsum = np.sum(np.stack(gs).astype(np.float64), axis=0)
        ref = o.compress(gsum, union, rows, cols, 9)
        ref.workers = W
        assert np.array_equal(host(m.table.table), ref.table.astype(np.float32))
        assert np.array_equal(host(s2.sparse_decompress(m)), o.decompress(ref).astype(np.float32))


def test_unbiasedness_over_seeds(s2):
    """Acceptance #5 / Theorem csmean: r=3, lambda=0.5 — the per-index mean error of
    the median query over fresh sketch seeds is within 4 standard errors of 0."""
    import torch

    rng = np.random.default_rng(21)
    d = 4000
    g = np.zeros(d, np.float32)
    nzi = rng.choice(d, 400, replace=False)
    g[nzi] = rng.standard_normal(400).astype(np.float32)
    cols = o.sketch_cols(0.5, 0.1, d, 3)
    probes = nzi[:40]
    gt = cuda(g)
    trials = 3000
    ests = torch.empty(trials, probes.size, device="cuda")
    pr = cuda(probes.astype(np.int64))
    for t in range(trials):
        p = s2.sparse_compress(gt, None, 3, cols, int(o.derive_seed(7, t)), check_finite=False)
        ests[t] = s2.sparse_decompress(p)[pr]
    e = host(ests).astype(np.float64) - g[probes][None, :]
    mean = e.mean(0)
    se = e.std(0, ddof=1) / np.sqrt(trials)
    assert (np.abs(mean) <= 4 * se + 1e-12).all(), np.abs(mean / se).max()


def test_injective_identity(s2):
    """mask = all, r = 1, c = d injective -> payload decodes to g exactly."""
    g = np.random.default_rng(4).standard_normal(1000).astype(np.float32)
    p = s2.sparse_compress(cuda(g), None, 1, 1000, 0, injective=True)
    assert np.array_equal(host(s2.sparse_decompress(p)), g)
    with pytest.raises(ValueError, match="injective mapping requires indices < buckets"):
        s2.sparse_compress(cuda(g), None, 1, 10, 0, injective=True)


def test_wire_roundtrip(s2):
    g = o.synthetic_gradient(50_000, 0.02, 0, kind="int")
    p = s2.sparse_compress(cuda(g), None, 3, 331, 77)
    data = p.to_bytes()
    ref = o.compress(g, g != 0, 3, 331, 77)
    assert data == ref.to_bytes()
    q = s2.sparse_payload_from_bytes(data)
    assert np.array_equal(words_u32(q.mask.words), words_u32(p.mask.words))
    assert np.array_equal(host(q.table.table), host(p.table.table))
    assert q.alpha == p.alpha


def test_compressor_plugin_nonzero(s2):
    """SparseSketchCompressor protocol (sparse.py:288-323) driven like casq.ef_step (casq.py:315-332)."""
    d = 20_000
    comp = s2.SparseSketchCompressor(d, d, 200, mask="nonzero")
    assert comp.mergeable and comp.name == "sparse" and comp.prepare(None) is None
    g = o.synthetic_gradient(d, 0.01, 0, kind="int")
    pay = comp.compress(cuda(g))
    est = comp.decompress(comp.merge([pay]))
    ref = o.decompress(o.compress(g, g != 0, 3, comp.cols, 0))
    assert np.array_equal(host(est), ref.astype(np.float32))
    assert comp.payload_nbytes(pay) == 53 + (d + 7) // 8 + 4 * 3 * comp.cols


def test_host_pipeline(s2):
    """HostPipeline: pinned host gradients in, host results out, copies overlapped across steps."""
    import torch

    from paper_2110_02140_b200.reducer import HostPipeline

    d = 1_000_003
    red = s2.S2Reducer(d, rows=3, cols=7919, seed=3)
    pipe = HostPipeline(red)
    gs = [o.synthetic_gradient(d, a, k, kind="int") for k, a in enumerate((0.01, 0.03, 0.002, 0.01, 0.05))]
    hin = [torch.from_numpy(g).pin_memory() for g in gs]
    hout = [torch.empty(d, dtype=torch.float32).pin_memory() for _ in gs]
    for gi, go in zip(hin, hout):
        pipe.submit(gi, go)
    pipe.drain()
    for g, go in zip(gs, hout):
        ref = o.decompress(o.compress(g, g != 0, 3, 7919, 3))
        assert np.array_equal(go.numpy(), ref.astype(np.float32))


def test_block_topk_golden_and_random(s2):
    """GPU block_topk (sparse.py:70-80) against the live-reference fixture and the oracle."""
    z = load("s2_blocks_topk")
    for w in range(int(z["W"])):
        m = s2.block_topk(cuda(z["grads"][w]), 333, 40)
        assert np.array_equal(words_u32(m.words), z["words"][w])
    rng = np.random.default_rng(8)
    for d, nb, k in ((10_000, 100, 7), (4097, 4097, 300), (100_000, 5000, 1), (100_000, 5000, 5000),
                     (1_000_003, 7919, 250), (33, 5, 2)):
        g = (rng.standard_normal(d) * (rng.random(d) < 0.5)).astype(np.float32)
        m = s2.block_topk(cuda(g), nb, k)
        assert np.array_equal(m.flags, o.block_topk(g, nb, k)), (d, nb, k)
        assert int(m.flags.sum()) == k


def test_block_topk_ties_lower_index(s2):
    """SPEC.md:425 tight case: equal block energies -> ties broken by the lower block index."""
    g = np.ones(16, np.float32)
    assert s2.block_topk(cuda(g), 4, 1).flags.tolist() == [True, False, False, False]
    g = np.tile(np.array([1.0, -2.0], np.float32), 40)
    assert s2.block_topk(cuda(g), 8, 3).flags.tolist() == [True, True, True] + [False] * 5
    g = np.zeros(100, np.float32)  # all-zero norms: the first k blocks
    assert np.array_equal(s2.block_topk(cuda(g), 10, 4).flags, o.block_topk(g, 10, 4))
    with pytest.raises(ValueError, match=r"k must be in \[1, 10\], got 11"):
        s2.block_topk(cuda(g), 10, 11)


def test_compressor_plugin_topk(s2):
    """SparseSketchCompressor with the reference's default block Top-K mask vs the oracle."""
    rng = np.random.default_rng(9)
    d, nb, k = 50_000, 500, 25
    comp = s2.SparseSketchCompressor(d, nb, k)
    g = (rng.integers(-100, 100, d) * (rng.random(d) < 0.3)).astype(np.float32)
    pay = comp.compress(cuda(g))
    flags = o.block_topk(g, nb, k)
    assert np.array_equal(pay.mask.flags, flags)
    ref = o.compress(g, flags, 3, comp.cols, 0)
    assert np.array_equal(host(pay.table.table), ref.table.astype(np.float32))
    assert pay.alpha == ref.alpha
    assert np.array_equal(host(comp.decompress(comp.merge([pay]))), o.decompress(ref).astype(np.float32))


def test_graphed_reduce(s2):
    """CUDA-graph replay (two captured phases) gives the same results as direct reduces."""
    import torch

    from paper_2110_02140_b200.reducer import GraphedReduce

    d = 1_000_000
    red = s2.S2Reducer(d, rows=3, cols=16384, seed=0)
    g_static = torch.zeros(d, device="cuda")
    out_static = torch.empty(d, device="cuda")
    gr = GraphedReduce(red, g_static, out_static)
    for k, alpha in enumerate((0.01, 0.03, 0.002, 0.02, 0.01)):
        g = o.synthetic_gradient(d, alpha, 10 + k, kind="int")
        g_static.copy_(torch.from_numpy(g))
        gr()
        ref = o.decompress(o.compress(g, g != 0, 3, 16384, 0))
        assert np.array_equal(host(out_static), ref.astype(np.float32)), k


def test_random_shapes_bit_exact(s2):
    """Fuzz: random dims (ragged tiles and words), block counts, rows 1..16, non-power-of-two and
    tiny widths, 64-bit seeds, W = 1..5 and densities, integer values (every cell sum < 2^24) —
    bitmaps, merged tables and decodes bit-exact against the oracle through the functional API."""
    rng = np.random.default_rng(2110)
    for trial in range(40):
        dim = int(rng.integers(1, 300_000))
        nb = dim if rng.random() < 0.6 else int(rng.integers(1, dim + 1))
        rows = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 16]))
        W = int(rng.integers(1, 6))
        dens = float(rng.choice([0.0005, 0.01, 0.1, 0.5]))
        nnz = max(1, int(dens * dim))
        cols = max(1, int(rng.integers(max(1, W * nnz // 8000), max(2, W * nnz // 8000) + 5000)))
        seed = int(rng.integers(0, 2**63))
        grads = []
        for w in range(W):
            g = np.zeros(dim, np.float32)
            pos = rng.choice(dim, min(nnz, dim), replace=False)
            v = rng.integers(-1000, 1001, pos.size).astype(np.float32)
            v[v == 0] = 1.0
            g[pos] = v
            grads.append(g)
        ps = [s2.sparse_compress(cuda(g), None, rows, cols, seed, num_blocks=nb) for g in grads]
        ops = [o.compress(g, o.nonzero_flags(g, nb), rows, cols, seed) for g in grads]
        for p, q in zip(ps, ops):
            assert np.array_equal(words_u32(p.mask.words)[: o.mask_words(q.flags).size], o.mask_words(q.flags)), trial
            assert np.array_equal(host(p.table.table), q.table.astype(np.float32)), trial
        m, om = s2.sparse_merge(ps), o.merge(ops)
        assert np.array_equal(host(m.table.table), om.table.astype(np.float32)), trial
        out = host(s2.sparse_decompress(m))
        assert np.array_equal(out, o.decompress(om).astype(np.float32)), (trial, dim, nb, rows, cols, W)


def test_injective_decompress_rejects_out_of_range(s2):
    """Injective mapping with cols < dim (core.py:131-135): a block mask whose selected coordinates
    reach past cols raises the reference's ValueError at decompress (the query maps every selected
    coordinate, zeros included, sparse.py:211-213) instead of reading past the table."""
    d = 1000
    g = np.zeros(d, np.float32)
    g[[3, 7]] = [1.0, 2.0]
    part = s2.BlockPartition(d, 10)  # 100-element blocks
    ok = s2.sparse_compress(cuda(g), s2.BlockMask(part, [True] + [False] * 9), 1, 100, 0, injective=True)
    assert np.array_equal(host(s2.sparse_decompress(ok))[:100], g[:100])
    bad = s2.sparse_compress(cuda(g), s2.BlockMask(part, [True, True] + [False] * 8), 1, 150, 0, injective=True)
    with pytest.raises(ValueError, match="injective mapping requires indices < buckets"):
        s2.sparse_decompress(bad)


def test_sparsify_topk_delta_golden(s2):
    """sparsify / topk_delta_check (sparse.py:217-242) against the live-reference fixture."""
    z = load("topk_delta")
    for (d, nb, k), g, sp, chk in zip(z["params"], z["grads"], z["sparsified"], z["checks"]):
        out = host(s2.sparsify(cuda(g[:d]), int(nb), int(k)))
        assert np.array_equal(out, sp[:d].astype(np.float32))
        kept, bound = s2.topk_delta_check(cuda(g[:d]), int(nb), int(k))
        assert bound == chk[1] and abs(kept - chk[0]) <= 1e-12 and kept >= bound


def test_block_topk_near_ties(s2):
    """Blocks holding permutations of the same values have equal norms in exact arithmetic; the
    GPU's float64 norm (warp-shuffle order) and np.linalg.norm (BLAS order) may round such near-
    ties differently.  Every block whose reference norm is separated from the k-th norm by more
    than 8 ulp must agree; only blocks inside that band may swap (documented in DESIGN.md §5)."""
    rng = np.random.default_rng(31)
    for trial in range(20):
        nb, bs = int(rng.integers(50, 400)), int(rng.integers(3, 200))
        base = rng.standard_normal(bs).astype(np.float32)
        g = np.concatenate([rng.permutation(base) * (1.0 if rng.random() < 0.7 else rng.random() * 2)
                            for _ in range(nb)]).astype(np.float32)
        k = int(rng.integers(1, nb))
        got = s2.block_topk(cuda(g), nb, k).flags
        ref = o.block_topk(g, nb, k)
        norms = np.array([np.linalg.norm(g[b * bs:(b + 1) * bs].astype(np.float64)) for b in range(nb)])
        kth = np.sort(norms)[::-1][k - 1]
        band = np.abs(norms - kth) <= 8 * np.spacing(kth)
        assert int(got.sum()) == k
        assert np.array_equal(got[~band], ref[~band]), trial


def test_back_to_back_reduces_overlap(s2):
    """Reduces launched back to back with no host sync (the compress of reduce i+1 overlaps the
    decode of reduce i through the period-4 buffer rotation), then every output checked; and a
    reduce whose input IS the previous output (the compress must then wait for that decode)."""
    import torch

    d = 1_000_003
    red = s2.S2Reducer(d, rows=3, cols=16384, seed=0)
    gs = [o.synthetic_gradient(d, a, 40 + k, kind="int") for k, a in enumerate([0.01, 0.03, 0.002, 0.05] * 3)]
    gt = [cuda(g) for g in gs]
    outs = [torch.empty(d, device="cuda") for _ in gs]
    for g, out in zip(gt, outs):
        red.reduce(g, out=out)
    torch.cuda.synchronize()
    for k, (g, out) in enumerate(zip(gs, outs)):
        ref = o.decompress(o.compress(g, g != 0, 3, 16384, 0))
        assert np.array_equal(host(out), ref.astype(np.float32)), k
    # chained: out1 = reduce(g); out2 = reduce(out1) with no sync in between
    g = gs[0]
    o1 = red.reduce(gt[0])
    o2 = red.reduce(o1)
    r1 = o.decompress(o.compress(g, g != 0, 3, 16384, 0)).astype(np.float32)
    r2 = o.decompress(o.compress(r1, r1 != 0, 3, 16384, 0)).astype(np.float32)
    assert np.array_equal(host(o1), r1) and np.array_equal(host(o2), r2)
    red.check()


def test_reduce_many_single_gpu(s2):
    """reduce_many at W = 1 equals sequential reduces, including a batch whose input aliases an
    earlier output of the batch (sequential fallback)."""
    import torch

    d = 300_007
    red = s2.S2Reducer(d, rows=3, cols=4099, seed=1)
    gs = [o.synthetic_gradient(d, 0.02, k, kind="int") for k in range(5)]
    outs = red.reduce_many([cuda(g) for g in gs])
    for g, out in zip(gs, outs):
        assert np.array_equal(host(out), o.decompress(o.compress(g, g != 0, 3, 4099, 1)).astype(np.float32))
    a = torch.empty(d, device="cuda")
    b = torch.empty(d, device="cuda")
    red.reduce_many([cuda(gs[0]), a], outs=[a, b])  # step 1 reads step 0's output
    r0 = o.decompress(o.compress(gs[0], gs[0] != 0, 3, 4099, 1)).astype(np.float32)
    r1 = o.decompress(o.compress(r0, r0 != 0, 3, 4099, 1)).astype(np.float32)
    assert np.array_equal(host(a), r0) and np.array_equal(host(b), r1)
    red.check()
