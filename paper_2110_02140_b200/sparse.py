"""S2 Reducer sparse-sketch compress / merge / decompress on B200.

Drop-in mirror of /root/reference/pkg/src/sketchgrad/sparse.py: the same
public names, argument meanings and ValueError messages, on CUDA float32
tensors.  Every computation runs in libs2.so (sm_100a kernels); this module
only shapes arguments and allocates outputs.

Differences from the reference, all deliberate and documented in DESIGN.md:
  * tensors are CUDA float32 (the reference computes in float64 and ships
    float32 on the wire, sparse.py:129); results agree within the fp32
    tolerance of DESIGN.md §Parity, bit-exactly for bitmaps/indices/hashes;
  * ``sparse_compress`` accepts ``mask=None`` (or ``"nonzero"``) to build the
    non-zero bitmap inside the compress kernel (the north-star mask rule,
    PAPER.md:263), equivalent to ``BlockMask(part, g != 0)``;
  * ``SparsePayload.alpha`` / ``size_ratio`` are computed lazily from device
    counters so that compress never blocks the host.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import (S2_CNT_NNZ, S2_CNT_NONFINITE, S2_CNT_SELECTED, S2_MASK_GIVEN, S2_MASK_NONZERO,
                   S2_NUM_COUNTERS, check, lib, ptr, stream_ptr)
from .core import BlockPartition, as_gradient
from .sketch import CountSketchTable, get_plan

MAGIC = b"S2SK"  # sparse.py:25
WIRE_VERSION = 1  # sparse.py:26
DEFAULT_ROWS = 3  # sparse.py:27
DEFAULT_SIZE_RATIO = 0.5  # sparse.py:28


def _words_for(num_blocks: int) -> int:
    return -(-num_blocks // 32)


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _new_counters(device) -> torch.Tensor:
    return torch.zeros(S2_NUM_COUNTERS, dtype=torch.int64, device=device)


class BlockMask:
    """Bitmap over a block partition, held on the GPU as little-endian uint32 words
    (sparse.py:31-61).  Bit k of word w flags block 32w+k."""

    def __init__(self, partition: BlockPartition, flags=None, *, words: torch.Tensor | None = None, device=None):
        self.partition = partition
        nwords = _words_for(partition.num_blocks)
        if words is not None:
            if words.numel() != nwords:
                raise ValueError("flag count must equal the block count")
            self.words = words
            return
        f = flags.detach().cpu().numpy() if isinstance(flags, torch.Tensor) else np.asarray(flags)
        f = f.astype(bool).reshape(-1)
        if f.size != partition.num_blocks:
            raise ValueError("flag count must equal the block count")  # sparse.py:40-41
        raw = np.packbits(f.astype(np.uint8), bitorder="little").tobytes()
        raw += b"\x00" * (4 * nwords - len(raw))
        host = torch.from_numpy(np.frombuffer(raw, dtype="<i4").copy())
        self.words = host.to(device or _device())

    # -- reference API ---------------------------------------------------
    @property
    def flags(self) -> np.ndarray:
        """Host bool[num_blocks] copy of the bitmap (the reference's ``flags`` field)."""
        raw = self.words.detach().cpu().numpy().astype("<i4").tobytes()
        return np.unpackbits(np.frombuffer(raw, np.uint8), count=self.partition.num_blocks,
                             bitorder="little").astype(bool)

    def selected_indices(self) -> torch.Tensor:
        """Ascending int64 coordinates inside set blocks (sparse.py:44-49), compacted on the GPU."""
        return _compact(self, None)[0]

    def selected_fraction(self) -> float:
        """Fraction of coordinates inside selected blocks (sparse.py:51-53)."""
        p = self.partition
        plan = get_plan(p.dim, p.num_blocks, 1, 1, 0)
        cnt = _new_counters(self.words.device)
        check(lib.s2_selected_count(plan.handle, ptr(self.words), ptr(cnt), stream_ptr()), "selected_count")
        return float(int(cnt[S2_CNT_SELECTED])) / p.dim

    def union(self, other: "BlockMask") -> "BlockMask":
        if self.partition != other.partition:
            raise ValueError("incompatible payloads: field 'partition' differs")  # sparse.py:56-57
        return _union([self, other])

    def to_bytes(self) -> bytes:
        """packbits little-endian (sparse.py:60-61): the device words, trimmed."""
        raw = self.words.detach().cpu().numpy().astype("<i4").tobytes()
        return raw[: -(-self.partition.num_blocks // 8)]

    def __eq__(self, other) -> bool:
        return (isinstance(other, BlockMask) and self.partition == other.partition
                and torch.equal(self.words, other.words))


def _union(masks) -> BlockMask:
    part = masks[0].partition
    stacked = torch.stack([m.words for m in masks])
    out = torch.empty_like(masks[0].words)
    check(lib.s2_bitmap_or(out.numel(), ptr(stacked), len(masks), ptr(out), stream_ptr()), "union")
    return BlockMask(part, words=out)


def _compact(mask: BlockMask, g: torch.Tensor | None):
    """Ordered compaction on the GPU: a counting pass sizes the outputs exactly, then the write pass."""
    p = mask.partition
    plan = get_plan(p.dim, p.num_blocks, 1, 1, 0)
    dev = mask.words.device
    scratch = torch.empty(int(lib.s2_compact_scratch_bytes(plan.handle)) // 8 + 1, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib.s2_compact(plan.handle, ptr(mask.words), ptr(g), None, None, ptr(count), ptr(scratch), stream_ptr()),
          "compact(count)")
    n = int(count.item())
    idx = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    vals = torch.empty(max(n, 1), dtype=torch.float32, device=dev) if g is not None else None
    check(lib.s2_compact(plan.handle, ptr(mask.words), ptr(g), ptr(idx), ptr(vals), ptr(count), ptr(scratch),
                         stream_ptr()), "compact")
    return idx[:n], (vals[:n] if vals is not None else None)


def mask_from_bytes(data: bytes, partition: BlockPartition) -> BlockMask:
    """sparse.py:64-67."""
    raw = np.frombuffer(data, dtype=np.uint8)
    flags = np.unpackbits(raw, count=partition.num_blocks, bitorder="little").astype(bool)
    return BlockMask(partition, flags)


def nonzero_mask(g, num_blocks: int | None = None) -> BlockMask:
    """BlockMask whose flags mark blocks holding a non-zero, built by the compress kernel."""
    g = as_gradient(g)
    p = BlockPartition(g.numel(), num_blocks or g.numel())
    return sparse_compress(g, None, 1, 1, 0, num_blocks=p.num_blocks, check_finite=True).mask


def block_topk(g, num_blocks: int, k: int) -> BlockMask:
    """Select the k blocks of largest L2 norm, ties to the lower block index (sparse.py:70-80).

    float64 block norms + an 8-pass radix select with a stable tie-break, on the GPU
    (csrc/s2_topk.cu)."""
    g = as_gradient(g)
    partition = BlockPartition(g.numel(), num_blocks)
    if not 1 <= k <= num_blocks:
        raise ValueError(f"k must be in [1, {num_blocks}], got {k}")
    if not bool(torch.isfinite(g).all()):
        raise ValueError("gradient vector contains NaN or Inf")  # as_gradient, core.py:157-158
    plan = get_plan(partition.dim, num_blocks, 1, 1, 0)
    scratch = torch.empty(int(lib.s2_block_topk_scratch_bytes(plan.handle)) // 8 + 1, dtype=torch.int64,
                          device=g.device)
    words = torch.empty(_words_for(num_blocks), dtype=torch.int32, device=g.device)
    check(lib.s2_block_topk(plan.handle, ptr(g), int(k), ptr(words), ptr(scratch), stream_ptr()), "block_topk")
    return BlockMask(partition, words=words)


def sketch_cols(size_ratio: float, alpha: float, dim: int, rows: int = DEFAULT_ROWS) -> int:
    """Columns per row so rows*cols ~= size_ratio*alpha*dim cells (sparse.py:83-88)."""
    if size_ratio <= 0:
        raise ValueError("size_ratio must be positive")
    cells = size_ratio * alpha * dim
    return max(1, -(-int(np.ceil(cells)) // rows))


@dataclass
class SparsePayload:
    """Bitmap plus signed sketch of the values inside selected blocks (sparse.py:91-129).

    ``alpha`` and ``size_ratio`` are read from device counters on first access.
    """

    mask: BlockMask
    table: CountSketchTable
    _alpha: float | None = None
    _size_ratio: float | None = None
    workers: int = 1
    counters: torch.Tensor | None = field(default=None, repr=False)

    @property
    def alpha(self) -> float:
        if self._alpha is None:
            if self.counters is not None:
                self._alpha = float(int(self.counters[S2_CNT_SELECTED])) / self.mask.partition.dim
            else:
                self._alpha = self.mask.selected_fraction()
        return self._alpha

    @property
    def size_ratio(self) -> float:
        if self._size_ratio is None:
            a = self.alpha
            self._size_ratio = self.table.rows * self.table.cols / (a * self.mask.partition.dim) if a > 0 else float("inf")
        return self._size_ratio

    def selected_count(self) -> int:
        """Coordinates inside selected blocks, sizes()[flags].sum() (sparse.py:51-53, :273)."""
        if self.counters is not None:
            return int(self.counters[S2_CNT_SELECTED])
        p = self.mask.partition
        plan = get_plan(p.dim, p.num_blocks, 1, 1, 0)
        cnt = _new_counters(self.mask.words.device)
        check(lib.s2_selected_count(plan.handle, ptr(self.mask.words), ptr(cnt), stream_ptr()), "selected_count")
        return int(cnt[S2_CNT_SELECTED])

    @property
    def nnz(self) -> int:
        """Values inserted into the sketch (device counter)."""
        return int(self.counters[S2_CNT_NNZ]) if self.counters is not None else -1

    def compat_key(self) -> dict:
        return {"partition": self.mask.partition, "sketch_params": self.table.params()}  # sparse.py:105-109

    def serialized_nbytes(self) -> int:
        bitmap_nbytes = -(-self.mask.partition.num_blocks // 8)
        return 4 + 1 + 6 * 8 + bitmap_nbytes + 4 * self.table.rows * self.table.cols  # sparse.py:111-113

    def to_bytes(self) -> bytes:
        """S2SK wire (sparse.py:115-129)."""
        if self.table.injective:
            raise ValueError("injective payloads have no wire representation")
        p = self.mask.partition
        header = struct.pack("<4sBQQQQQQ", MAGIC, WIRE_VERSION, p.dim, p.num_blocks, self.table.rows,
                             self.table.cols, self.table.seed & 0xFFFFFFFFFFFFFFFF, 0)
        return header + self.mask.to_bytes() + self.table.table.detach().cpu().numpy().astype("<f4").tobytes()


def sparse_payload_from_bytes(data: bytes, device=None) -> SparsePayload:
    """sparse.py:132-148."""
    if len(data) < 5 or data[:4] != MAGIC:
        raise ValueError("not a sparse payload (bad magic)")
    if data[4] != WIRE_VERSION:
        raise ValueError(f"unsupported sparse wire version {data[4]}")
    dim, blocks, rows, cols, seed, _ = struct.unpack_from("<QQQQQQ", data, 5)
    off = 5 + 48
    partition = BlockPartition(dim, blocks)
    nb = -(-blocks // 8)
    mask = mask_from_bytes(data[off: off + nb], partition)
    off += nb
    table = CountSketchTable(rows, cols, seed, dim, device=device)
    flat = np.frombuffer(data, dtype="<f4", count=rows * cols, offset=off)
    table.table.copy_(torch.from_numpy(flat.copy()).reshape(rows, cols))
    return SparsePayload(mask, table)


def _raise_nonfinite(counters: torch.Tensor) -> None:
    if int(counters[S2_CNT_NONFINITE]):
        raise ValueError("gradient vector contains NaN or Inf")  # core.py:157-158


def sparse_compress(g, mask: BlockMask | str | None, rows: int, cols: int, seed: int,
                    injective: bool = False, *, num_blocks: int | None = None,
                    check_finite: bool = True) -> SparsePayload:
    """Insert every non-zero entry of the selected blocks into a fresh signed sketch
    (sparse.py:151-171) — one fused kernel: bitmap + compaction + sketch insert.

    ``mask``: a BlockMask (used as given), or None / "nonzero" to build the
    non-zero bitmap over ``num_blocks`` blocks (default: one block per element).
    ``check_finite``: synchronise and raise ValueError on NaN/Inf like the
    reference's as_gradient; False keeps the call fully asynchronous (the flag
    stays readable in ``payload.counters``).
    """
    g = as_gradient(g)
    d = g.numel()
    if isinstance(mask, BlockMask):
        if d != mask.partition.dim:
            raise ValueError(f"dimension mismatch: mask dim {mask.partition.dim}, vector {d}")  # sparse.py:159-162
        part = mask.partition
        mode = S2_MASK_GIVEN
        words = mask.words
    elif mask is None or mask == "nonzero":
        part = BlockPartition(d, num_blocks or d)
        mode = S2_MASK_NONZERO
        words = torch.empty(_words_for(part.num_blocks), dtype=torch.int32, device=g.device)
    else:
        raise ValueError(f"unknown mask {mask!r}")
    table = CountSketchTable(rows, cols, seed, d, injective=injective, device=g.device)
    plan = get_plan(d, part.num_blocks, rows, cols, seed, injective)
    counters = _new_counters(g.device)
    if injective and cols < d:
        # HashMapping(injective) raises if any inserted index >= buckets (core.py:131-135)
        probe = BlockMask(part, words=words) if mode == S2_MASK_GIVEN else None
        if probe is not None:
            idx, vals = _compact(probe, g)
            if idx.numel() and int(idx[-1]) >= cols:
                raise ValueError("injective mapping requires indices < buckets")
        else:
            nz = torch.nonzero(g).reshape(-1)
            if nz.numel() and int(nz[-1]) >= cols:
                raise ValueError("injective mapping requires indices < buckets")
    check(lib.s2_compress(plan.handle, ptr(g), ptr(words), ptr(table.table), mode, ptr(counters), stream_ptr()),
          "compress")
    if check_finite:
        _raise_nonfinite(counters)
    out_mask = mask if mode == S2_MASK_GIVEN else BlockMask(part, words=words)
    return SparsePayload(out_mask, table, counters=counters)


def compacted_values(g, mask: BlockMask):
    """The (indices, values) pairs sparse_compress inserts (sparse.py:164-168): ascending
    non-zero coordinates inside set blocks, compacted on the GPU."""
    g = as_gradient(g)
    if g.numel() != mask.partition.dim:
        raise ValueError(f"dimension mismatch: mask dim {mask.partition.dim}, vector {g.numel()}")
    return _compact(mask, g)


def sparse_merge(payloads) -> SparsePayload:
    """OR the bitmaps, sum the sketch tables, re-derive alpha and lambda (sparse.py:174-196)."""
    payloads = list(payloads)
    if not payloads:
        raise ValueError("nothing to merge")
    ref = payloads[0].compat_key()
    for p in payloads[1:]:
        key = p.compat_key()
        for name, value in ref.items():
            if key[name] != value:
                raise ValueError(f"incompatible payloads: field {name!r} differs ({value!r} vs {key[name]!r})")
    t0 = payloads[0].table
    if len(payloads) == 1:
        mask = payloads[0].mask
        table = t0
    else:
        mask = _union([p.mask for p in payloads])
        table = CountSketchTable(t0.rows, t0.cols, t0.seed, t0.dim, t0.injective, device=t0.device)
        stacked = torch.stack([p.table.table for p in payloads])
        check(lib.s2_table_sum(t0.rows * t0.cols, ptr(stacked), len(payloads), ptr(table.table), stream_ptr()),
              "merge")
    return SparsePayload(mask, table, workers=sum(p.workers for p in payloads))


def sparse_decompress(payload: SparsePayload, workers: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Query every selected index and divide by the worker count; zeros elsewhere (sparse.py:199-214)."""
    if workers is None:
        workers = payload.workers
    if workers < 1:
        raise ValueError("workers must be >= 1")
    p = payload.mask.partition
    t = payload.table
    if t.injective and t.cols < p.dim:
        # the query maps every selected coordinate, zeros inside set blocks included
        # (sparse.py:211-213); HashMapping(injective) raises for any index >= buckets (core.py:133-134)
        sel = np.flatnonzero(payload.mask.flags)
        if sel.size and min((int(sel[-1]) + 1) * p.block_size, p.dim) - 1 >= t.cols:
            raise ValueError("injective mapping requires indices < buckets")
    plan = get_plan(p.dim, p.num_blocks, t.rows, t.cols, t.seed, t.injective)
    if out is None:
        out = torch.empty(p.dim, dtype=torch.float32, device=t.device)
    check(lib.s2_decode(plan.handle, ptr(payload.mask.words), ptr(t.table), int(workers), ptr(out), stream_ptr()),
          "decompress")
    return out


def sparsify(g, num_blocks: int, k: int) -> torch.Tensor:
    """g with every block outside the top-k (by L2 norm) zeroed (sparse.py:217-224), on the GPU."""
    g = as_gradient(g)
    idx = block_topk(g, num_blocks, k).selected_indices()
    out = torch.zeros_like(g)
    out[idx] = g[idx]
    return out


def topk_delta_check(g, num_blocks: int, k: int) -> tuple[float, float]:
    """Energy kept by block top-k versus the k/b floor (sparse.py:227-242): (kept_ratio, bound);
    the ratio is 1 for the zero vector.  Norms accumulate in float64 like the reference."""
    g = as_gradient(g)
    bound = k / num_blocks
    g64 = g.double()
    total = float(g64 @ g64)
    if total == 0.0:
        return 1.0, bound
    kept = sparsify(g, num_blocks, k).double()
    return float(kept @ kept) / total, bound


@dataclass
class CommCost:
    """Wire cost of one payload against dense and coordinate baselines (sparse.py:244-261)."""

    payload_bits: int
    dense_bits: int
    coordinate_bits: int
    value_bits: int
    bitmap_bits: int
    header_bits: int

    @property
    def ratio_vs_dense(self) -> float:
        return self.payload_bits / self.dense_bits

    @property
    def ratio_vs_coordinate(self) -> float:
        return self.payload_bits / self.coordinate_bits


def sparse_comm_bits(payload: SparsePayload) -> CommCost:
    """Account the payload's bits: bitmap + 32-bit table cells + header (sparse.py:264-285).
    The coordinate baseline sends each selected value as 32 bits plus a ceil(log2 dim)-bit
    index; the selected count comes from the compress kernel's device counter."""
    part = payload.mask.partition
    nnz = payload.selected_count()
    index_bits = max(1, (part.dim - 1).bit_length())
    return CommCost(
        payload_bits=8 * payload.serialized_nbytes(),
        dense_bits=32 * part.dim,
        coordinate_bits=nnz * (32 + index_bits),
        value_bits=32 * payload.table.rows * payload.table.cols,
        bitmap_bits=part.num_blocks,
        header_bits=8 * (4 + 1 + 6 * 8),
    )


class SparseSketchCompressor:
    """Block-mask + signed-sketch compressor plugin (sparse.py:288-323).

    Same protocol as the reference (mergeable, name, prepare, compress, merge,
    decompress, payload_nbytes).  ``mask="topk"`` (the reference default) runs the
    GPU block Top-K; ``mask="nonzero"`` selects the north-star non-zero bitmap.
    """

    mergeable = True
    name = "sparse"

    def __init__(self, dim: int, num_blocks: int, topk_blocks: int, rows: int = DEFAULT_ROWS,
                 size_ratio: float = DEFAULT_SIZE_RATIO, seed: int = 0, injective: bool = False,
                 mask: str = "topk"):
        self.dim = dim
        self.num_blocks = num_blocks
        self.topk_blocks = topk_blocks
        self.rows = rows
        self.size_ratio = size_ratio
        self.seed = seed
        self.injective = injective
        self.mask_mode = mask
        alpha = BlockPartition(dim, num_blocks).sizes()[:topk_blocks].sum() / dim  # sparse.py:304-305
        self.cols = sketch_cols(size_ratio, float(alpha), dim, rows)

    def prepare(self, reference, step: int = 0):
        return None  # stateless between iterations (sparse.py:307-308)

    def compress(self, values) -> SparsePayload:
        if self.mask_mode == "nonzero":
            return sparse_compress(values, None, self.rows, self.cols, self.seed, injective=self.injective,
                                   num_blocks=self.num_blocks)
        mask = block_topk(values, self.num_blocks, self.topk_blocks)
        return sparse_compress(values, mask, self.rows, self.cols, self.seed, injective=self.injective)

    def merge(self, payloads) -> SparsePayload:
        return sparse_merge(payloads)

    def decompress(self, payload) -> torch.Tensor:
        return sparse_decompress(payload)

    def payload_nbytes(self, payload) -> int:
        return payload.serialized_nbytes()
