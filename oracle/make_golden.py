"""Generate golden vectors for the S2 path by running the LIVE reference — test infrastructure.

Usage (in the build container, where /root/reference exists):

    python oracle/make_golden.py            # writes tests/golden/*.npz

Everything written here comes from ``sketchgrad`` itself
(/root/reference/pkg/src/sketchgrad: core.py, sketch.py, sparse.py), imported
read-only via sys.path — never from ``oracle/s2_oracle.py``, so the fixtures pin
the oracle rather than the other way round.  The GPU box has no
/root/reference; the committed .npz files travel instead.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import sketchgrad.core as core  # noqa: E402
    import sketchgrad.sketch as sketch  # noqa: E402
    import sketchgrad.sparse as sparse  # noqa: E402
    return core, sketch, sparse


def _grad(dim, alpha, rank, kind, base_seed=1234):
    # same recipe as oracle.synthetic_gradient, restated so the fixture does not
    # depend on the oracle module
    rng = np.random.default_rng(base_seed + rank)
    nnz = int(round(alpha * dim))
    pos = rng.choice(dim, nnz, replace=False)
    if kind == "normal":
        vals = rng.standard_normal(nnz).astype(np.float32)
        vals[vals == 0] = 1.0
    elif kind == "int":
        vals = rng.integers(-1000, 1001, size=nnz).astype(np.float32)
        vals[vals == 0] = 1.0
    elif kind == "subint":
        # fp32 subnormals: integers in units of 2^-149 (every partial sum stays subnormal and exact)
        k = rng.integers(-1000, 1001, size=nnz).astype(np.float64)
        k[k == 0] = 1.0
        vals = (k * 2.0 ** -149).astype(np.float32)
    elif kind == "underflow":
        # just above the normal range (+-[1, 1.5] x 2^-126): cells of opposite signs cancel into
        # the subnormal range, which a flush-to-zero accumulation would lose
        k = rng.integers(2 ** 23, 2 ** 23 + 2 ** 22, size=nnz).astype(np.float64)
        k *= rng.integers(0, 2, size=nnz) * 2.0 - 1.0
        vals = (k * 2.0 ** -149).astype(np.float32)
    else:
        raise ValueError(kind)
    g = np.zeros(dim, dtype=np.float32)
    g[pos] = vals
    return g


def _words(flags):
    raw = np.packbits(np.asarray(flags, np.uint8), bitorder="little").tobytes()
    raw += b"\x00" * ((-len(raw)) % 4)
    return np.frombuffer(raw, "<u4").copy()


def hash_kat(core):
    seeds = [0, 1, 42, 12345, 0xFFFFFFFFFFFFFFFF, 0x8000000000000000]
    js = list(range(8))
    ds = np.array([[core.derive_seed(s, j) for j in js] for s in seeds], dtype=np.uint64)
    rng = np.random.default_rng(7)
    idx = np.concatenate([
        np.arange(0, 64), np.array([999_999, 25_599_999, 109_999_999, 199_999_999, 354_999_999,
                                    2**31 - 1, 2**31, 2**32 - 2]),
        rng.integers(0, 2**32 - 1, size=1000),
    ]).astype(np.int64)
    cols_list = [1, 2, 3, 7, 8, 1000, 1667, 8334, 16384, 262144, 1_000_000, 1_048_576,
                 4_194_304, 2**31 - 1, 3_000_000_019]
    row_seeds = np.array([core.derive_seed(0, j) for j in range(5)] +
                         [core.derive_seed(42, j) for j in range(3)], dtype=np.uint64)
    words = np.stack([core._hash_words(np.uint64(s), idx) for s in row_seeds])
    buckets = np.stack([np.stack([core.hash_buckets(np.uint64(s), idx, c) for c in cols_list])
                        for s in row_seeds])
    signs = np.stack([core.hash_signs(np.uint64(s), idx) for s in row_seeds])
    mix_in = np.array([0, 1, 2, 0xFFFFFFFFFFFFFFFF, 0x243F6A8885A308D3], dtype=np.uint64)
    np.savez_compressed(
        os.path.join(OUT, "hash_kat.npz"),
        derive_seeds_in=np.array(seeds, dtype=np.uint64), derive_j=np.array(js), derive_out=ds,
        mix_in=mix_in, mix_out=core.mix64(mix_in),
        idx=idx, cols=np.array(cols_list, dtype=np.int64), row_seeds=row_seeds,
        words=words, buckets=buckets.astype(np.uint32), signs=signs,
    )


def tiny(sketch):
    t = sketch.CountSketchTable(3, 8, seed=0, dim=16)
    t.insert([1, 5, 9], [1.0, -2.0, 0.5])
    np.savez_compressed(os.path.join(OUT, "tiny_table.npz"), table=t.table,
                        query=t.query([1, 5, 9]))


def case(core, sparse, name, dim, alpha, rows, cols, W, kind, num_blocks=None, seed=0,
         topk=None, extra=None):
    """W workers: compress each with the non-zero (or top-k) mask, merge, decompress."""
    part = core.BlockPartition(dim, num_blocks or dim)
    grads, payloads = [], []
    for w in range(W):
        g = _grad(dim, alpha, w, kind) if extra is None else extra[w]
        g64 = g.astype(np.float64)
        if topk is not None:
            mask = sparse.block_topk(g64, part.num_blocks, topk)
        elif part.num_blocks == dim:
            mask = sparse.BlockMask(part, g64 != 0)
        else:
            bs = part.block_size
            flags = np.array([np.any(g64[s] != 0) for s in part.slices()])
            mask = sparse.BlockMask(part, flags)
        p = sparse.sparse_compress(g64, mask, rows, cols, seed)
        grads.append(g)
        payloads.append(p)
    m = sparse.sparse_merge(payloads)
    out = sparse.sparse_decompress(m)
    union_idx = m.mask.selected_indices()
    # L1 mass of every merged cell (tolerance scale)
    l1 = np.zeros((rows, cols))
    for g, p in zip(grads, payloads):
        idx = p.mask.selected_indices()
        v = g.astype(np.float64)[idx]
        nz = v != 0
        for j, rm in enumerate(m.table.row_maps):
            np.add.at(l1[j], rm.bucket(idx[nz]), np.abs(v[nz]))
    d = dict(
        dim=dim, num_blocks=part.num_blocks, rows=rows, cols=cols, seed=seed, W=W,
        grads=np.stack(grads),
        words=np.stack([_words(p.mask.flags) for p in payloads]),
        tables=np.stack([p.table.table for p in payloads]),
        alphas=np.array([p.alpha for p in payloads]),
        ratios=np.array([p.size_ratio for p in payloads]),
        union_words=_words(m.mask.flags), merged_table=m.table.table,
        merged_alpha=m.alpha, merged_ratio=m.size_ratio, merged_workers=m.workers,
        union_idx=union_idx, decode_at_union=out[union_idx],
        decode_nonzero_outside_union=int(np.count_nonzero(np.delete(out, union_idx))),
        l1_mass=l1,
        nbytes=payloads[0].serialized_nbytes(),
        wire_sha256=np.frombuffer(hashlib.sha256(payloads[0].to_bytes()).digest(), np.uint8),
        wire_head=np.frombuffer(payloads[0].to_bytes()[:53], np.uint8),
        # CommCost of worker 0's payload and of the merged payload (sparse.py:244-285)
        comm_bits=_comm(sparse.sparse_comm_bits(payloads[0])),
        comm_bits_merged=_comm(sparse.sparse_comm_bits(m)),
    )
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)


def topk_delta(sparse):
    """sparsify / topk_delta_check (sparse.py:217-242) on a few block layouts."""
    rng = np.random.default_rng(5)
    gs, outs, checks, params = [], [], [], []
    for d, nb, k in ((10_007, 100, 7), (4096, 4096, 300), (1000, 7, 3)):
        g = (rng.standard_normal(d) * (rng.random(d) < 0.3)).astype(np.float32)
        gs.append(np.pad(g, (0, 10_007 - d)))
        outs.append(np.pad(sparse.sparsify(g.astype(np.float64), nb, k), (0, 10_007 - d)))
        checks.append(sparse.topk_delta_check(g.astype(np.float64), nb, k))
        params.append((d, nb, k))
    np.savez_compressed(os.path.join(OUT, "topk_delta.npz"), grads=np.stack(gs), sparsified=np.stack(outs),
                        checks=np.array(checks), params=np.array(params))


def _comm(c):
    return np.array([c.payload_bits, c.dense_bits, c.coordinate_bits, c.value_bits, c.bitmap_bits, c.header_bits],
                    dtype=np.int64)


def main():
    core, sketch, sparse = _ref()
    os.makedirs(OUT, exist_ok=True)
    hash_kat(core)
    tiny(sketch)
    topk_delta(sparse)
    # configs[0]: the oracle case, 1M / 99% / 3x16384 / W=1
    case(core, sparse, "s2_1m_w1", 1_000_000, 0.01, 3, 16384, 1, "normal")
    # mergeability (acceptance #7) at W=2,4,8; non-pow2 cols
    case(core, sparse, "s2_int_w8", 200_000, 0.01, 3, sparse.sketch_cols(0.5, 0.08, 200_000), 8, "int")
    case(core, sparse, "s2_normal_w4", 300_001, 0.02, 3, 5000, 4, "normal")
    case(core, sparse, "s2_normal_w2_r5", 100_003, 0.05, 5, 1000, 2, "normal")
    # even row counts: lower median (sketch.py:117-128)
    case(core, sparse, "s2_r2", 20_000, 0.05, 2, 97, 3, "normal")
    case(core, sparse, "s2_r4", 20_000, 0.05, 4, 101, 3, "int")
    case(core, sparse, "s2_r1", 5_000, 0.1, 1, 64, 2, "normal")
    # block-granular bitmap (b < d), ragged last block and empty tail blocks (core.py:172-211)
    case(core, sparse, "s2_blocks_nz", 10_007, 0.003, 3, 211, 3, "normal", num_blocks=1000)
    case(core, sparse, "s2_blocks_topk", 10_007, 0.2, 3, 500, 2, "normal", num_blocks=333, topk=40)
    # edge cases: d not a multiple of 32, -0.0, all-zero worker, d = 1
    g_edge = np.zeros(37, np.float32)
    g_edge[[0, 5, 31, 32, 36]] = [1.5, -2.0, 3.0, -0.0, 7.25]
    case(core, sparse, "s2_edge37", 37, 0.0, 3, 5, 2, "normal",
         extra=[g_edge, np.zeros(37, np.float32)])
    case(core, sparse, "s2_d1", 1, 0.0, 3, 2, 1, "normal", extra=[np.array([-3.0], np.float32)])
    # fp32 subnormal and underflowing values (the reference adds in float64, sketch.py:111)
    case(core, sparse, "s2_subnormal_int", 30_011, 0.05, 3, 97, 3, "subint")
    case(core, sparse, "s2_underflow", 20_000, 0.1, 3, 53, 2, "underflow")
    print("golden written to", os.path.abspath(OUT))


if __name__ == "__main__":
    main()
