"""CPU: pin the oracle (oracle/s2_oracle.py) against golden vectors made by the live reference.

The fixtures in tests/golden were produced by oracle/make_golden.py importing
/root/reference/pkg/src/sketchgrad itself.  When the reference is present (the
build container) the oracle is additionally cross-checked against it live.
"""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import s2_oracle as o

REF = "/root/reference/pkg/src"
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "s2_*.npz")))


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def test_appendix_b_kats():
    # SURVEY.md Appendix B, taken from the live oracle during the survey
    assert o.row_seeds(0, 5) == [0xA8871E3718CA0053, 0x74D28E025CEAAC29, 0x890710CED7FBC4AF,
                                 0xFC4729067514681E, 0x3B6F9CEFDB22F673]
    assert o.row_seeds(42, 3) == [0xCA4A76AE36B1E15B, 0xF4034FB65ACC0D70, 0x5A5EDE7975EC7488]
    assert int(o.mix64(0)) == 0 and int(o.mix64(1)) == 0x5692161D100B05E5
    s0 = o.row_seeds(0, 1)[0]
    assert [int(w) for w in o.hash_words(s0, [0, 1, 2])] == [0xBB90C7A6337C19D9, 0x2319836A87853061,
                                                             0x65684F19BD20F47F]
    idx = [0, 1, 2, 3, 999999, 25599999, 354999999]
    assert o.hash_buckets(s0, idx, 16384).tolist() == [6617, 12385, 13439, 13822, 8440, 2701, 3647]
    assert o.hash_buckets(s0, idx, 1667).tolist() == [202, 799, 771, 133, 926, 446, 1490]
    assert o.hash_buckets(s0, idx, 1000000).tolist() == [352345, 669025, 460031, 496766, 955448, 573709, 451135]
    assert o.hash_signs(s0, idx).tolist() == [-1, 1, 1, -1, -1, 1, 1]
    assert o.sketch_cols(0.5, 0.01, 1e6) == 1667 and o.sketch_cols(0.5, 0.05, 1e6) == 8334


def test_hash_kat_golden():
    z = load("hash_kat")
    for si, s in enumerate(z["derive_seeds_in"]):
        for jj, j in enumerate(z["derive_j"]):
            assert o.derive_seed(int(s), int(j)) == int(z["derive_out"][si, jj])
    assert np.array_equal(o.mix64(z["mix_in"]), z["mix_out"])
    for si, s in enumerate(z["row_seeds"]):
        assert np.array_equal(o.hash_words(s, z["idx"]), z["words"][si])
        assert np.array_equal(o.hash_signs(s, z["idx"]), z["signs"][si])
        for ci, c in enumerate(z["cols"]):
            assert np.array_equal(o.hash_buckets(s, z["idx"], int(c)), z["buckets"][si, ci].astype(np.int64))


def test_tiny_table():
    z = load("tiny_table")
    t = np.zeros((3, 8))
    o.sketch_insert(t, o.row_seeds(0, 3), [1, 5, 9], [1.0, -2.0, 0.5], 8)
    assert np.array_equal(t, z["table"])
    assert np.array_equal(o.sketch_query(t, o.row_seeds(0, 3), [1, 5, 9], 8), z["query"])
    assert z["query"].tolist() == [1.0, -2.0, 0.5]


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_golden(name):
    z = load(name)
    dim, nb, rows, cols, seed, W = (int(z[k]) for k in ("dim", "num_blocks", "rows", "cols", "seed", "W"))
    payloads = []
    for w in range(W):
        g = z["grads"][w]
        if name == "s2_blocks_topk":
            flags = o.words_to_flags(z["words"][w], nb)
            assert np.array_equal(flags, o.block_topk(g, nb, 40))
        else:
            flags = o.nonzero_flags(g, nb)
        assert np.array_equal(o.mask_words(flags), z["words"][w])
        p = o.compress(g, flags, rows, cols, seed)
        assert np.array_equal(p.table, z["tables"][w])  # bit-identical float64
        assert p.alpha == z["alphas"][w]
        payloads.append(p)
    m = o.merge(payloads)
    assert np.array_equal(o.mask_words(m.flags), z["union_words"])
    assert np.array_equal(m.table, z["merged_table"])
    assert m.alpha == float(z["merged_alpha"]) and m.workers == int(z["merged_workers"])
    out = o.decompress(m)
    idx = o.selected_indices(m.flags, dim)
    assert np.array_equal(idx, z["union_idx"])
    assert np.array_equal(out[idx], z["decode_at_union"])
    assert np.count_nonzero(np.delete(out, idx)) == int(z["decode_nonzero_outside_union"]) == 0
    assert payloads[0].serialized_nbytes() == int(z["nbytes"])
    import hashlib

    wire = payloads[0].to_bytes()
    assert np.array_equal(np.frombuffer(wire[:53], np.uint8), z["wire_head"])
    assert hashlib.sha256(wire).digest() == z["wire_sha256"].tobytes()
    assert list(o.comm_bits(payloads[0])) == z["comm_bits"].tolist()  # sparse.py:264-285
    assert list(o.comm_bits(m)) == z["comm_bits_merged"].tolist()


def test_sparsify_topk_delta_golden():
    z = load("topk_delta")
    for (d, nb, k), g, sp, chk in zip(z["params"], z["grads"], z["sparsified"], z["checks"]):
        assert np.array_equal(o.sparsify(g[:d], int(nb), int(k)), sp[:d])
        assert o.topk_delta_check(g[:d], int(nb), int(k)) == tuple(chk)


def test_as_shipped_restatement():
    """The loop-for-loop restatement bench.py times as the as-shipped reference equals the oracle."""
    for W, d, nb in ((1, 20_000, 20_000), (3, 30_011, 30_011)):
        grads = [o.synthetic_gradient(d, 0.02, r) for r in range(W)]
        ref = o.decompress(o.merge([o.compress(g, g != 0, 3, 97, 5) for g in grads]))
        assert np.array_equal(o.reduce_as_shipped(grads, 3, 97, 5), ref)
    f = np.random.default_rng(0).random(1000) < 0.3
    assert np.array_equal(o.selected_indices_as_shipped(f, 9_999), o.selected_indices(f, 9_999))


def test_edge_semantics():
    z = load("s2_edge37")
    # -0.0 at index 32 is not a non-zero (sparse.py:167); all-zero worker has an empty mask
    f = o.nonzero_flags(z["grads"][0], 37)
    assert not f[32] and f[[0, 5, 31, 36]].all()
    assert not o.nonzero_flags(z["grads"][1], 37).any()


def test_oracle_errors():
    with pytest.raises(ValueError, match="NaN or Inf"):
        o.as_gradient([1.0, np.nan])
    with pytest.raises(ValueError, match="at least one entry"):
        o.as_gradient([])
    with pytest.raises(ValueError, match="workers must be >= 1"):
        o.decompress(o.compress(np.ones(4), np.ones(4, bool), 3, 4, 0), workers=0)
    with pytest.raises(ValueError, match="nothing to merge"):
        o.merge([])


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted (GPU box)")
def test_oracle_vs_live_reference_random():
    """Cross-check the restatement against the as-shipped reference on fresh random cases."""
    import sys

    sys.path.insert(0, REF)
    import sketchgrad.core as rc
    import sketchgrad.sparse as rs

    rng = np.random.default_rng(99)
    for trial in range(6):
        d = int(rng.integers(1, 3000))
        nb = int(rng.integers(1, d + 1))
        rows = int(rng.integers(1, 6))
        cols = int(rng.integers(1, 300))
        seed = int(rng.integers(0, 2**63))
        W = int(rng.integers(1, 5))
        gs = [(rng.standard_normal(d) * (rng.random(d) < 0.1)).astype(np.float32) for _ in range(W)]
        part = rc.BlockPartition(d, nb)
        refp = []
        for g in gs:
            flags = np.array([np.any(g.astype(np.float64)[s] != 0) for s in part.slices()])
            refp.append(rs.sparse_compress(g, rs.BlockMask(part, flags), rows, cols, seed))
        rm = rs.sparse_merge(refp)
        ours = o.merge([o.compress(g, o.nonzero_flags(g, nb), rows, cols, seed) for g in gs])
        assert np.array_equal(ours.flags, rm.mask.flags)
        assert np.array_equal(ours.table, rm.table.table)
        assert np.array_equal(o.decompress(ours), rs.sparse_decompress(rm))


def test_bench_generator_matches_oracle_recipe():
    """bench.py draws its inputs with paper_2110_02140_b200.synthetic (the product may not import
    oracle/); the numpy recipe must produce the oracle's bytes."""
    from paper_2110_02140_b200 import synthetic

    for d, a, r in ((10_000, 0.01, 0), (100_003, 0.05, 3)):
        assert np.array_equal(synthetic.numpy_gradient(d, a, r), o.synthetic_gradient(d, a, r))


@pytest.mark.parametrize("d,nb,W", [(50_003, 50_003, 1), (50_003, 50_003, 3), (40_000, 400, 2)])
def test_parallel_reference_matches_oracle(d, nb, W):
    """bench.py's reference arm (oracle/parallel.py, chunked over worker processes) computes the
    oracle's reduce; on small-integer inputs the float64 sums are exact in any order."""
    from oracle.parallel import ParallelReference

    gs = [o.synthetic_gradient(d, 0.02, r, kind="int") for r in range(W)]
    _, ref = o.reduce(gs, nb, 3, 512, 7)
    pr = ParallelReference(gs, 3, 512, 7, procs=3, num_blocks=nb)
    try:
        for _ in range(2):  # second step reuses the shared buffers
            out = pr.step().copy()
            assert np.array_equal(out, ref)
    finally:
        pr.close()
