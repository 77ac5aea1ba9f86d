"""Multi-core CPU reference reduce for bench.py's reference arm — TEST INFRASTRUCTURE ONLY.

The oracle restatement (s2_oracle.py) is single-threaded NumPy, as is the reference.
To time the CPU path "with all the host threads it can use", this module splits the
same arithmetic over coordinate chunks in a persistent process pool with shared
memory: each worker runs the oracle's compress on its chunk into its own float64
partial table; the parent sums the partials (and the ranks' tables, OR-ing the
flags — sparse_merge, sparse.py:174-196); workers then run the oracle's decompress
query (lower median, /W) on their chunks of the union.  Only the summation order of
the float64 table differs from the single-threaded oracle.
"""

from __future__ import annotations

import os
from multiprocessing import get_context, shared_memory

import numpy as np

from . import s2_oracle as o

_S = {}  # worker-side attached arrays


def _attach(spec):
    out = {}
    for name, (shm_name, shape, dtype) in spec.items():
        shm = shared_memory.SharedMemory(name=shm_name)
        out[name] = (shm, np.ndarray(shape, dtype=dtype, buffer=shm.buf))
    return out


def _init(spec, rows, cols, seed, bs):
    _S.update(_attach(spec))
    _S["cfg"] = (rows, cols, seed, o.row_seeds(seed, rows))
    _S["bs"] = bs


def _compress_chunk(args):
    rank, k, lo, hi = args
    rows, cols, seed, seeds = _S["cfg"]
    g = _S["grads"][1][rank, lo:hi].astype(np.float64)
    flags = g != 0.0
    bs = _S["bs"]
    if bs > 1:  # block flag = block holds a non-zero; chunks are block-aligned (nonzero_flags)
        nb = -(-flags.size // bs)
        pad = np.zeros(nb * bs, dtype=bool)
        pad[: flags.size] = flags
        flags = np.repeat(pad.reshape(nb, bs).any(axis=1), bs)[: flags.size]
    _S["flags"][1][rank, lo:hi] = flags
    idx = np.flatnonzero(flags)
    t = _S["partial"][1][rank, k]
    t[:] = 0.0
    if idx.size:
        o.sketch_insert(t, seeds, idx + lo, g[idx], cols)
    return int(idx.size)


def _decode_chunk(args):
    lo, hi, workers = args
    rows, cols, seed, seeds = _S["cfg"]
    union = _S["union"][1][lo:hi]
    out = _S["out"][1]
    out[lo:hi] = 0.0
    idx = np.flatnonzero(union) + lo
    if idx.size:
        out[idx] = o.sketch_query(_S["table"][1], seeds, idx, cols) / workers
    return int(idx.size)


class ParallelReference:
    """W ranks' gradients reduced on the host with `procs` worker processes."""

    def __init__(self, grads, rows, cols, seed=0, procs=None, num_blocks=None):
        self.W = len(grads)
        self.d = grads[0].size
        self.rows, self.cols, self.seed = rows, cols, seed
        self.procs = procs or os.cpu_count() or 1
        self.nchunks = self.procs
        bs = o.block_size(self.d, num_blocks or self.d)
        nblk = -(-self.d // bs)
        bounds = np.minimum(np.linspace(0, nblk, self.nchunks + 1).astype(np.int64) * bs, self.d)
        self.chunks = [(int(bounds[i]), int(bounds[i + 1])) for i in range(self.nchunks)]
        self._shm = []

        def make(name, shape, dtype):
            nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
            shm = shared_memory.SharedMemory(create=True, size=max(nbytes, 1))
            self._shm.append(shm)
            spec[name] = (shm.name, shape, np.dtype(dtype).str)
            return np.ndarray(shape, dtype=dtype, buffer=shm.buf)

        spec = {}
        gr = make("grads", (self.W, self.d), np.float32)
        for r, g in enumerate(grads):
            gr[r] = g
        make("flags", (self.W, self.d), np.bool_)
        self.partial = make("partial", (self.W, self.nchunks, rows, cols), np.float64)
        self.union = make("union", (self.d,), np.bool_)
        self.table = make("table", (rows, cols), np.float64)
        self.out = make("out", (self.d,), np.float64)
        self.flags = np.ndarray((self.W, self.d), dtype=np.bool_, buffer=self._shm[1].buf)
        self.pool = get_context("fork").Pool(self.procs, initializer=_init, initargs=(spec, rows, cols, seed, bs))

    def step(self) -> np.ndarray:
        jobs = [(r, k, lo, hi) for r in range(self.W) for k, (lo, hi) in enumerate(self.chunks)]
        self.pool.map(_compress_chunk, jobs)
        # sparse_merge: sum every rank's partial tables, OR the flags
        np.sum(self.partial.reshape(-1, self.rows, self.cols), axis=0, out=self.table)
        np.logical_or.reduce(self.flags, axis=0, out=self.union)
        self.pool.map(_decode_chunk, [(lo, hi, self.W) for lo, hi in self.chunks])
        return self.out

    def close(self):
        self.pool.close()
        self.pool.join()
        for shm in self._shm:
            shm.close()
            shm.unlink()
