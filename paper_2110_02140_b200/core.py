"""Shared primitives of the S2 path: seeded hashing and block partitions.

Mirrors /root/reference/pkg/src/sketchgrad/core.py (names, arguments, errors).
Hashing is evaluated by libs2.so (the same device code the kernels inline,
compiled for the host); there is no NumPy re-implementation on the product
path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib

MASK64 = 0xFFFFFFFFFFFFFFFF


def mix64(x):
    """splitmix64 finalizer (core.py:27-38); scalar or array -> uint64."""
    arr = np.asarray(x, dtype=np.uint64)
    out = np.fromiter((lib.s2_mix64(int(v)) for v in arr.reshape(-1)), dtype=np.uint64, count=arr.size)
    return out.reshape(arr.shape) if arr.ndim else np.uint64(out[0])


def derive_seed(*parts) -> int:
    """Fold integer parts into one 64-bit seed (core.py:44-54)."""
    buf = (ctypes.c_uint64 * max(1, len(parts)))(*[int(p) & MASK64 for p in parts])
    return int(lib.s2_derive_seed(buf, len(parts)))


def row_seeds(seed: int, rows: int) -> list[int]:
    """derive_seed(seed, j) for every sketch row (sketch.py:96-99)."""
    out = (ctypes.c_uint64 * rows)()
    check(lib.s2_row_seeds(int(seed) & MASK64, rows, out))
    return [int(v) for v in out]


def _hash(seed: int, indices, buckets: int):
    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.int64).reshape(-1))
    b = np.empty(idx.size, dtype=np.int64)
    s = np.empty(idx.size, dtype=np.int8)
    check(lib.s2_hash_host(int(seed) & MASK64, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), idx.size,
                           int(buckets), b.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                           s.ctypes.data_as(ctypes.POINTER(ctypes.c_int8))))
    return b, s, np.shape(indices)


def hash_buckets(seed: int, indices, buckets: int):
    """(w & (2^63-1)) % buckets (core.py:89-100)."""
    if buckets < 1:
        raise ValueError(f"buckets must be >= 1, got {buckets}")
    b, _, shape = _hash(seed, indices, buckets)
    return b.reshape(shape)


def hash_signs(seed: int, indices):
    """1 - 2*(w >> 63) as float64 (core.py:103-106)."""
    _, s, shape = _hash(seed, indices, 1)
    return s.astype(np.float64).reshape(shape)


@dataclass(frozen=True)
class BlockPartition:
    """Contiguous partition of [0, dim) into num_blocks blocks of ceil(dim/num_blocks),
    ragged last block (core.py:172-211)."""

    dim: int
    num_blocks: int

    def __post_init__(self):
        if self.dim < 1:
            raise ValueError(f"dim must be >= 1, got {self.dim}")
        if not 1 <= self.num_blocks <= self.dim:
            raise ValueError(f"num_blocks must be in [1, dim={self.dim}], got {self.num_blocks}")

    @property
    def block_size(self) -> int:
        return -(-self.dim // self.num_blocks)

    def slices(self) -> list[slice]:
        size = self.block_size
        return [slice(min(b * size, self.dim), min((b + 1) * size, self.dim)) for b in range(self.num_blocks)]

    def sizes(self) -> np.ndarray:
        size = self.block_size
        starts = np.minimum(np.arange(self.num_blocks, dtype=np.int64) * size, self.dim)
        stops = np.minimum(starts + size, self.dim)
        return stops - starts

    def block_of(self, index: int) -> int:
        if not 0 <= index < self.dim:
            raise ValueError(f"index {index} outside [0, {self.dim})")
        return index // self.block_size


def as_gradient(values, device=None):
    """Validate a gradient and return it as a contiguous float32 CUDA vector (core.py:147-159).

    The reference upcasts to float64; this path computes in float32 (the
    reference's own wire precision, sparse.py:129).  NaN/Inf detection happens
    on the device inside the compress kernel (see ``sparse_compress``).
    """
    import torch

    if isinstance(values, torch.Tensor):
        t = values
    else:
        t = torch.as_tensor(np.asarray(values))
    t = t.reshape(-1)
    if t.numel() < 1:
        raise ValueError("gradient vector must have at least one entry")
    dev = device or (t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    t = t.to(device=dev, dtype=torch.float32)
    if not t.is_contiguous() or t.data_ptr() % 16:
        t = t.contiguous().clone()
    return t
