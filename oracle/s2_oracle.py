"""CPU oracle for the S2 Reducer sparse-sketch reduce path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The shipped path
(``paper_2110_02140_b200``) never routes through it.

It is a NumPy restatement of the reference algorithm in
``/root/reference/pkg/src/sketchgrad`` (core.py, sketch.py, sparse.py), with
every function citing the file:line it follows.  The only intentional change
from the as-shipped reference is index extraction: the reference builds
``BlockMask.selected_indices`` with a Python loop over ``BlockPartition.slices``
(sparse.py:44-49, core.py:195-200); here it is one vectorised expression.  The
arithmetic that produces every number (uint64 hashing, ``np.add.at`` float64
accumulation in ascending-index order, sort + lower median, ÷W) is the same
NumPy call sequence, so results are bit-identical (pinned in
``tests/test_oracle.py`` against fixtures generated from the live reference by
``oracle/make_golden.py``).

Parity pinned: yes — golden vectors in ``tests/golden/`` were produced by
importing the reference itself (see ``oracle/make_golden.py``).
"""

from __future__ import annotations

import struct

import numpy as np

# core.py:16-24 — the constants of the hash family.
MASK63 = np.uint64(0x7FFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX_1 = np.uint64(0xBF58476D1CE4E5B9)
MIX_2 = np.uint64(0x94D049BB133111EB)
DERIVE_INIT = np.uint64(0x243F6A8885A308D3)  # core.py:41

MAGIC = b"S2SK"  # sparse.py:25
WIRE_VERSION = 1  # sparse.py:26
DEFAULT_ROWS = 3  # sparse.py:27
DEFAULT_SIZE_RATIO = 0.5  # sparse.py:28


# ---------------------------------------------------------------- hashing


def mix64(x):
    """splitmix64 finalizer, wrapping mod 2^64 (core.py:27-38)."""
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * MIX_1
        z = (z ^ (z >> np.uint64(27))) * MIX_2
        return z ^ (z >> np.uint64(31))


def derive_seed(*parts) -> int:
    """Fold integer parts into one 64-bit seed (core.py:44-54)."""
    acc = DERIVE_INIT
    with np.errstate(over="ignore"):
        for part in parts:
            acc = mix64(acc + np.uint64(int(part) & 0xFFFFFFFFFFFFFFFF) * GOLDEN)
    return int(acc)


def row_seeds(seed: int, rows: int) -> list[int]:
    """Per-row seeds of a CountSketchTable: derive_seed(seed, j) (sketch.py:96-99)."""
    return [derive_seed(seed, j) for j in range(rows)]


def hash_words(seed, indices):
    """w = mix64(seed + (i+1)*G) (core.py:70-75)."""
    s = np.asarray(seed, dtype=np.uint64)
    idx = np.asarray(indices, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(s + (idx + np.uint64(1)) * GOLDEN)


def hash_buckets(seed, indices, buckets: int):
    """(w & (2^63-1)) % buckets (core.py:89-100)."""
    if buckets < 1:
        raise ValueError(f"buckets must be >= 1, got {buckets}")
    words = hash_words(seed, indices)
    return ((words & MASK63) % np.uint64(buckets)).astype(np.int64)


def hash_signs(seed, indices):
    """1 - 2*(w >> 63) as float64 (core.py:103-106)."""
    words = hash_words(seed, indices)
    return 1.0 - 2.0 * (words >> np.uint64(63)).astype(np.float64)


# ------------------------------------------------------ partitions / masks


def as_gradient(values) -> np.ndarray:
    """float64 flatten + validation (core.py:147-159)."""
    g = np.asarray(values, dtype=np.float64)
    if g.ndim != 1:
        g = g.reshape(-1)
    if g.size < 1:
        raise ValueError("gradient vector must have at least one entry")
    if not np.all(np.isfinite(g)):
        raise ValueError("gradient vector contains NaN or Inf")
    return g


def block_size(dim: int, num_blocks: int) -> int:
    """ceil(dim / num_blocks) (core.py:191-193)."""
    return -(-dim // num_blocks)


def block_sizes(dim: int, num_blocks: int) -> np.ndarray:
    """Per-block sizes with a ragged last block (core.py:202-206)."""
    size = block_size(dim, num_blocks)
    starts = np.minimum(np.arange(num_blocks, dtype=np.int64) * size, dim)
    stops = np.minimum(starts + size, dim)
    return stops - starts


def nonzero_flags(g, num_blocks: int) -> np.ndarray:
    """Block flag = block holds a non-zero (== block_topk(g, b, nnz-blocks)).

    For num_blocks == dim this is ``g != 0`` (−0.0 is a zero, sparse.py:167).
    """
    g = as_gradient(g)
    bs = block_size(g.size, num_blocks)
    nz = g != 0.0
    if bs == 1:
        return nz.copy()
    pad = np.zeros(num_blocks * bs, dtype=bool)
    pad[: g.size] = nz
    return pad.reshape(num_blocks, bs).any(axis=1)


def selected_indices(flags, dim: int) -> np.ndarray:
    """Ascending coordinates inside set blocks (sparse.py:44-49, vectorised)."""
    flags = np.asarray(flags, dtype=bool)
    bs = block_size(dim, flags.size)
    blocks = np.flatnonzero(flags)
    if blocks.size == 0:
        return np.zeros(0, dtype=np.int64)
    if bs == 1:
        return blocks.astype(np.int64)
    idx = (blocks[:, None] * bs + np.arange(bs)[None, :]).reshape(-1)
    return idx[idx < dim].astype(np.int64)


def selected_indices_as_shipped(flags, dim: int) -> np.ndarray:
    """The reference's own index extraction, restated loop for loop for timing the CPU path as
    shipped: BlockPartition.slices() builds one slice object per block
    (core.py:195-200) and selected_indices concatenates an arange per selected block
    (sparse.py:44-49).  Same result as ``selected_indices``; ~100x slower at b = d."""
    flags = np.asarray(flags, dtype=bool)
    nb = flags.size
    size = block_size(dim, nb)
    slices = [slice(min(b * size, dim), min((b + 1) * size, dim)) for b in range(nb)]
    picked = [np.arange(s.start, s.stop) for b, s in enumerate(slices) if flags[b]]
    if not picked:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate(picked).astype(np.int64)


def reduce_as_shipped(grads, rows: int, cols: int, seed: int) -> np.ndarray:
    """One W-rank reduce with the reference's call structure and element bitmap (b = d):
    per rank BlockMask(part, g != 0) + sparse_compress (sparse.py:151-171), sparse_merge as a
    left fold (:174-196), sparse_decompress (:199-214) — every index extraction through the
    as-shipped slice loop.  Timing only; results equal decompress(merge(compress(...)))."""
    seeds = row_seeds(seed, rows)
    dim = grads[0].size
    merged, flags_u, W = None, None, len(grads)
    for g in grads:
        g = as_gradient(g)
        flags = g != 0
        table = np.zeros((rows, cols), dtype=np.float64)
        idx = selected_indices_as_shipped(flags, dim)
        if idx.size:
            vals = g[idx]
            nz = vals != 0.0
            sketch_insert(table, seeds, idx[nz], vals[nz], cols)
        merged = table if merged is None else merged + table
        flags_u = flags if flags_u is None else flags_u | flags
    out = np.zeros(dim, dtype=np.float64)
    idx = selected_indices_as_shipped(flags_u, dim)
    if idx.size:
        out[idx] = sketch_query(merged, seeds, idx, cols) / W
    return out


def selected_fraction(flags, dim: int) -> float:
    """alpha = selected coordinates / dim (sparse.py:51-53)."""
    flags = np.asarray(flags, dtype=bool)
    return float(block_sizes(dim, flags.size)[flags].sum()) / dim


def mask_to_bytes(flags) -> bytes:
    """packbits little-endian (sparse.py:60-61)."""
    return np.packbits(np.asarray(flags, dtype=np.uint8), bitorder="little").tobytes()


def mask_words(flags) -> np.ndarray:
    """Bitmap as little-endian uint32 words: bit k of word w == flags[32w+k]."""
    raw = mask_to_bytes(flags)
    pad = (-len(raw)) % 4
    return np.frombuffer(raw + b"\x00" * pad, dtype="<u4").copy()


def words_to_flags(words, num_blocks: int) -> np.ndarray:
    raw = np.asarray(words, dtype="<u4").tobytes()
    return np.unpackbits(np.frombuffer(raw, np.uint8), count=num_blocks, bitorder="little").astype(bool)


def sketch_cols(size_ratio: float, alpha: float, dim: int, rows: int = DEFAULT_ROWS) -> int:
    """max(1, ceil(ceil(lambda*alpha*d)/r)) (sparse.py:83-88)."""
    if size_ratio <= 0:
        raise ValueError("size_ratio must be positive")
    cells = size_ratio * alpha * dim
    return max(1, -(-int(np.ceil(cells)) // rows))


def block_topk(g, num_blocks: int, k: int) -> np.ndarray:
    """Top-k blocks by L2 norm, ties to the lower index (sparse.py:70-80)."""
    g = as_gradient(g)
    if not 1 <= k <= num_blocks:
        raise ValueError(f"k must be in [1, {num_blocks}], got {k}")
    bs = block_size(g.size, num_blocks)
    norms = np.array(
        [np.linalg.norm(g[min(b * bs, g.size): min((b + 1) * bs, g.size)]) for b in range(num_blocks)]
    )
    order = np.argsort(-norms, kind="stable")
    flags = np.zeros(num_blocks, dtype=bool)
    flags[order[:k]] = True
    return flags


def sparsify(g, num_blocks: int, k: int) -> np.ndarray:
    """Zero everything outside the top-k blocks (sparse.py:217-224)."""
    g = as_gradient(g)
    flags = block_topk(g, num_blocks, k)
    out = np.zeros_like(g)
    idx = selected_indices(flags, g.size)
    out[idx] = g[idx]
    return out


def topk_delta_check(g, num_blocks: int, k: int) -> tuple:
    """(|sparsify(g)|^2 / |g|^2, k/b), 1 for the zero vector (sparse.py:227-242)."""
    g = as_gradient(g)
    bound = k / num_blocks
    total = float(g @ g)
    if total == 0.0:
        return 1.0, bound
    kept = sparsify(g, num_blocks, k)
    return float(kept @ kept) / total, bound


# ---------------------------------------------------------------- sketch


def sketch_insert(table, seeds, indices, values, cols: int):
    """Per row ``np.add.at(T[j], h_j(idx), s_j(idx)*vals)`` (sketch.py:102-112)."""
    idx = np.asarray(indices, dtype=np.int64)
    vals = np.asarray(values, dtype=np.float64)
    for j, s in enumerate(seeds):
        np.add.at(table[j], hash_buckets(s, idx, cols), hash_signs(s, idx) * vals)
    return table


def sketch_query(table, seeds, indices, cols: int) -> np.ndarray:
    """Lower median over rows of s_j(i)*T[j, h_j(i)] (sketch.py:114-128)."""
    idx = np.asarray(indices, dtype=np.int64)
    est = np.stack([hash_signs(s, idx) * table[j, hash_buckets(s, idx, cols)] for j, s in enumerate(seeds)])
    est.sort(axis=0)
    return est[(len(seeds) - 1) // 2]


def sketch_l1_mass(seeds, indices, values, cols: int) -> np.ndarray:
    """M[j, c] = sum |v| over contributions to cell (j, c): the fp32 tolerance scale."""
    m = np.zeros((len(seeds), cols), dtype=np.float64)
    idx = np.asarray(indices, dtype=np.int64)
    av = np.abs(np.asarray(values, dtype=np.float64))
    for j, s in enumerate(seeds):
        np.add.at(m[j], hash_buckets(s, idx, cols), av)
    return m


# ------------------------------------------------------- S2 reducer ops


class Payload:
    """Oracle-side SparsePayload (sparse.py:91-103): flags + float64 table + bookkeeping."""

    def __init__(self, dim, flags, table, rows, cols, seed, workers=1):
        self.dim = dim
        self.flags = np.asarray(flags, dtype=bool)
        self.table = table
        self.rows = rows
        self.cols = cols
        self.seed = seed
        self.workers = workers

    @property
    def alpha(self) -> float:
        return selected_fraction(self.flags, self.dim)

    @property
    def size_ratio(self) -> float:
        a = self.alpha
        return self.rows * self.cols / (a * self.dim) if a > 0 else float("inf")

    def serialized_nbytes(self) -> int:
        """sparse.py:111-113."""
        return 4 + 1 + 6 * 8 + (-(-self.flags.size // 8)) + 4 * self.rows * self.cols

    def to_bytes(self) -> bytes:
        """S2SK wire (sparse.py:115-129)."""
        header = struct.pack(
            "<4sBQQQQQQ", MAGIC, WIRE_VERSION, self.dim, self.flags.size,
            self.rows, self.cols, self.seed & 0xFFFFFFFFFFFFFFFF, 0,
        )
        return header + mask_to_bytes(self.flags) + self.table.astype("<f4").tobytes()


def compress(g, flags, rows: int, cols: int, seed: int) -> Payload:
    """sparse_compress (sparse.py:151-171): insert non-zero entries of set blocks."""
    g = as_gradient(g)
    flags = np.asarray(flags, dtype=bool)
    if rows < 1 or cols < 1:
        raise ValueError(f"rows and cols must be >= 1, got {rows}x{cols}")
    seeds = row_seeds(seed, rows)
    table = np.zeros((rows, cols), dtype=np.float64)
    idx = selected_indices(flags, g.size)
    if idx.size:
        vals = g[idx]
        nz = vals != 0.0
        sketch_insert(table, seeds, idx[nz], vals[nz], cols)
    return Payload(g.size, flags, table, rows, cols, seed)


def merge(payloads) -> Payload:
    """sparse_merge (sparse.py:174-196): OR the masks, sum the tables left to right."""
    payloads = list(payloads)
    if not payloads:
        raise ValueError("nothing to merge")
    p0 = payloads[0]
    flags = p0.flags.copy()
    table = p0.table.copy()
    for p in payloads[1:]:
        if (p.dim, p.flags.size) != (p0.dim, p0.flags.size):
            raise ValueError("incompatible payloads: field 'partition' differs")
        if (p.rows, p.cols, p.seed) != (p0.rows, p0.cols, p0.seed):
            raise ValueError("incompatible payloads: field 'sketch_params' differs")
        flags = flags | p.flags
        table = table + p.table
    return Payload(p0.dim, flags, table, p0.rows, p0.cols, p0.seed, sum(p.workers for p in payloads))


def decompress(payload: Payload, workers=None) -> np.ndarray:
    """sparse_decompress (sparse.py:199-214): query set coordinates, ÷W, zeros elsewhere."""
    if workers is None:
        workers = payload.workers
    if workers < 1:
        raise ValueError("workers must be >= 1")
    out = np.zeros(payload.dim, dtype=np.float64)
    idx = selected_indices(payload.flags, payload.dim)
    if idx.size:
        out[idx] = sketch_query(payload.table, row_seeds(payload.seed, payload.rows), idx, payload.cols) / workers
    return out


def comm_bits(payload: Payload) -> tuple:
    """sparse_comm_bits (sparse.py:264-285): (payload, dense, coordinate, value, bitmap, header) bits;
    the coordinate baseline is 32 bits + ceil(log2 dim) index bits per selected coordinate."""
    nb = payload.flags.size
    nnz = int(block_sizes(payload.dim, nb)[payload.flags].sum())
    index_bits = max(1, (payload.dim - 1).bit_length())
    return (8 * payload.serialized_nbytes(), 32 * payload.dim, nnz * (32 + index_bits),
            32 * payload.rows * payload.cols, nb, 8 * (4 + 1 + 6 * 8))


def reduce(grads, num_blocks, rows, cols, seed):
    """Whole-box reduce on W gradients with the non-zero mask rule (north-star path)."""
    ps = [compress(g, nonzero_flags(g, num_blocks), rows, cols, seed) for g in grads]
    m = merge(ps)
    return m, decompress(m)


# -------------------------------------------------------- synthetic data


def synthetic_gradient(dim: int, alpha: float, rank: int = 0, kind: str = "normal",
                       base_seed: int = 1234) -> np.ndarray:
    """fp32 gradient, zero except round(alpha*d) positions (SURVEY §8(d) synthetic inputs).

    Positions: ``default_rng(base_seed + rank).choice(d, nnz, replace=False)``.
    ``kind``: "normal" (standard normal), "int" (uniform ints in [-1000, 1000],
    zero redrawn as 1 — bit-exact fp32 check) or "lognormal" (verify.py:694-702).
    """
    rng = np.random.default_rng(base_seed + rank)
    nnz = int(round(alpha * dim))
    pos = rng.choice(dim, nnz, replace=False)
    if kind == "normal":
        vals = rng.standard_normal(nnz).astype(np.float32)
        vals[vals == 0] = 1.0
    elif kind == "int":
        vals = rng.integers(-1000, 1001, size=nnz).astype(np.float32)
        vals[vals == 0] = 1.0
    elif kind == "lognormal":
        mags = rng.lognormal(-3.0, 0.8, size=nnz)
        signs = rng.integers(0, 2, size=nnz) * 2.0 - 1.0
        vals = (mags * signs).astype(np.float32)
    else:
        raise ValueError(kind)
    g = np.zeros(dim, dtype=np.float32)
    g[pos] = vals
    return g
