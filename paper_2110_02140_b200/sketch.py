"""Signed count-sketch table on the GPU (the CountSketchTable half of S2).

Mirrors /root/reference/pkg/src/sketchgrad/sketch.py:83-139 (CountSketchTable)
and :199-222 (merge).  The table is a float32 [rows, cols] CUDA tensor; insert
and query run the sm_100a kernels of libs2.so.  CountMinArray / AveragedSketch
belong to the CASQ compressor and are out of scope.
"""

from __future__ import annotations

import ctypes
import functools
import struct

import torch

from ._lib import check, lib, ptr, stream_ptr

SKCH_MAGIC = b"SKCH"  # sketch.py:30
WIRE_VERSION = 1
_KIND_COUNT_SKETCH = 1  # sketch.py:33


class Plan:
    """Owns one ``s2_plan`` (BlockPartition + CountSketchTable parameters)."""

    def __init__(self, dim: int, num_blocks: int, rows: int, cols: int, seed: int, injective: bool = False):
        h = ctypes.c_void_p()
        check(lib.s2_plan_create(int(dim), int(num_blocks), int(rows), int(cols),
                                 int(seed) & 0xFFFFFFFFFFFFFFFF, int(bool(injective)), ctypes.byref(h)))
        self.handle = h
        self.dim, self.num_blocks, self.rows, self.cols = int(dim), int(num_blocks), int(rows), int(cols)
        self.seed, self.injective = int(seed), bool(injective)
        self.words = int(lib.s2_plan_bitmap_words(h))
        self.block_size = int(lib.s2_plan_block_size(h))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and lib is not None:
            lib.s2_plan_destroy(h)
            self.handle = None


@functools.lru_cache(maxsize=64)
def get_plan(dim: int, num_blocks: int, rows: int, cols: int, seed: int, injective: bool = False) -> Plan:
    return Plan(dim, num_blocks, rows, cols, seed, injective)


def _index_tensor(indices, dim: int, device) -> torch.Tensor:
    idx = indices if isinstance(indices, torch.Tensor) else torch.as_tensor(indices)
    idx = idx.reshape(-1).to(device=device, dtype=torch.int64).contiguous()
    if idx.numel() and (int(idx.min()) < 0 or int(idx.max()) >= dim):
        raise ValueError(f"index outside [0, {dim})")  # sketch.py:108-109
    return idx


class CountSketchTable:
    """rows x cols signed sketch with a lower-median query (sketch.py:83-139)."""

    def __init__(self, rows: int, cols: int, seed: int, dim: int, injective: bool = False, device=None):
        if rows < 1 or cols < 1:
            raise ValueError(f"rows and cols must be >= 1, got {rows}x{cols}")  # sketch.py:87-88
        if dim < 1:
            raise ValueError(f"dim must be >= 1, got {dim}")
        self.rows, self.cols, self.seed, self.dim, self.injective = int(rows), int(cols), int(seed), int(dim), bool(injective)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.table = torch.zeros(self.rows, self.cols, dtype=torch.float32, device=self.device)

    def _plan(self) -> Plan:
        return get_plan(self.dim, self.dim, self.rows, self.cols, self.seed, self.injective)

    def insert(self, indices, values) -> "CountSketchTable":
        """Add s_j(i)*v at T[j, h_j(i)] for every row (sketch.py:102-112); zero values are no-ops."""
        idx = _index_tensor(indices, self.dim, self.device)
        vals = values if isinstance(values, torch.Tensor) else torch.as_tensor(values)
        vals = vals.reshape(-1).to(device=self.device, dtype=torch.float32).contiguous()
        if idx.shape != vals.shape:
            raise ValueError("indices and values must have matching shapes")
        if self.injective and idx.numel() and int(idx.max()) >= self.cols:
            raise ValueError("injective mapping requires indices < buckets")  # core.py:133-134
        check(lib.s2_sketch_insert(self._plan().handle, ptr(idx), ptr(vals), idx.numel(), ptr(self.table),
                                   stream_ptr()), "insert")
        return self

    def query(self, indices) -> torch.Tensor:
        """Lower median over rows of s_j(i)*T[j, h_j(i)] (sketch.py:114-128)."""
        idx = _index_tensor(indices, self.dim, self.device)
        if self.injective and idx.numel() and int(idx.max()) >= self.cols:
            raise ValueError("injective mapping requires indices < buckets")
        out = torch.empty(idx.numel(), dtype=torch.float32, device=self.device)
        check(lib.s2_sketch_query(self._plan().handle, ptr(idx), idx.numel(), ptr(self.table), ptr(out),
                                  stream_ptr()), "query")
        return out

    def query_one(self, index: int) -> float:
        return float(self.query([index])[0])

    def params(self) -> tuple:
        return ("count-sketch", self.dim, self.rows, self.cols, self.seed, self.injective)  # sketch.py:133-134

    def to_bytes(self) -> bytes:
        """SKCH wire, count-sketch kind (sketch.py:136-139, :225-229)."""
        if self.injective:
            raise ValueError("injective sketches have no wire representation")
        header = struct.pack("<4sBB", SKCH_MAGIC, WIRE_VERSION, _KIND_COUNT_SKETCH) + struct.pack(
            "<QQQQ", self.dim, self.rows, self.cols, self.seed & 0xFFFFFFFFFFFFFFFF)
        return header + self.table.detach().cpu().numpy().astype("<f4").tobytes()


def merge(a: CountSketchTable, b: CountSketchTable) -> CountSketchTable:
    """Parameter-checked element-wise sum into a new sketch (sketch.py:199-222)."""
    if type(a) is not type(b):
        raise ValueError(f"cannot merge {type(a).__name__} with {type(b).__name__}")
    if a.params() != b.params():
        raise ValueError(f"incompatible sketch parameters: {a.params()} vs {b.params()}")
    out = CountSketchTable(a.rows, a.cols, a.seed, a.dim, a.injective, device=a.device)
    stacked = torch.stack([a.table, b.table])
    check(lib.s2_table_sum(a.rows * a.cols, ptr(stacked), 2, ptr(out.table), stream_ptr()), "merge")
    return out
