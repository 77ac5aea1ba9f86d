"""Distributed S2 reduce: one process per GPU, NCCL over NVLink inside libs2.so.

This replaces the reference's in-process ``sparse_merge`` list fold
(sparse.py:174-196) with a real box-wide exchange:

    compress (K1+K2, local)  ->  sketch all-reduce + bitmap all-gather/OR (K3)
                             ->  decode (K4, replicated on every rank, ÷W)

``S2Reducer.reduce(g)`` is one C call (``s2_reduce``) on the caller's CUDA
stream; no host synchronisation happens inside it, so it can be captured in
a CUDA graph.  The NCCL communicator is created once from a unique id that
rank 0 broadcasts through torch.distributed (any backend).
"""

from __future__ import annotations

import ctypes

import torch

from ._lib import (S2_CNT_NNZ, S2_CNT_NONFINITE, S2_COMM_IPC, S2_COMM_NCCL, S2_NUM_COUNTERS, S2_STATUS_EXCHANGE,
                   S2_STATUS_NONFINITE, check, lib, ptr, stream_ptr)
from .core import as_gradient
from .sketch import Plan
from .sparse import DEFAULT_ROWS, DEFAULT_SIZE_RATIO, sketch_cols


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """Rank 0 of ``group`` creates the NCCL unique id; every rank returns the same 128 bytes
    (torch.distributed object broadcast; works over gloo or nccl)."""
    import torch.distributed as dist

    uid = (ctypes.c_uint8 * 128)()
    if rank == 0:
        check(lib.s2_nccl_unique_id(uid), "nccl unique id")
    box = [bytes(uid)]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(box, src=src, group=group)
    return box[0]


_STATUS_RING = 8  # outstanding reduces whose status words are checked without synchronising


class _StatusRing:
    """Per-reduce health words written by the decode kernel into mapped pinned host memory
    (s2_plan_set_status), checked once the reduce's event has completed — the previous
    steps' NaN/Inf and exchange-timeout flags surface without a host synchronisation."""

    def __init__(self, handle, device):
        self.h = handle
        self.words = torch.zeros(_STATUS_RING, dtype=torch.int32, pin_memory=True)
        self.pending = []  # (event, slot, phase-tag)
        self.n = 0
        self.device = device

    def arm(self) -> int:
        if len(self.pending) >= _STATUS_RING:  # the GPU lags by a full ring: wait for the oldest
            self.pending[0][0].synchronize()
            self.poll()
        k = self.n % _STATUS_RING
        self.n += 1
        self.words[k] = 0  # the decodes OR their error bits in
        check(lib.s2_plan_set_status(self.h, ctypes.c_void_p(self.words.data_ptr() + 4 * k)), "set status")
        return k

    def launched(self, k: int, stream) -> None:
        ev = torch.cuda.Event()
        ev.record(stream)
        self.pending.append((ev, k))

    def poll(self, wait: bool = False) -> None:
        while self.pending and (wait or self.pending[0][0].query()):
            ev, k = self.pending.pop(0)
            if wait:
                ev.synchronize()
            st = int(self.words[k]) & 0xFFFFFFFF
            if st & S2_STATUS_EXCHANGE:
                self.pending.clear()
                raise RuntimeError("S2 exchange: a cross-rank barrier timed out (a rank died, stalled past the "
                                   "timeout, or the ranks' reduce sequences diverged); the averaged gradient "
                                   "was set to NaN")
            if st & S2_STATUS_NONFINITE:
                self.pending.clear()
                raise ValueError("gradient vector contains NaN or Inf")  # core.py:157-158


class S2Reducer:
    """Averaged sparse-sketch all-reduce of a flat float32 gradient.

    Parameters mirror ``SparseSketchCompressor`` (sparse.py:294-305): ``cols``
    defaults to ``sketch_cols(size_ratio, alpha, dim, rows)``; ``num_blocks``
    defaults to ``dim`` (element bitmap, the north-star mask rule).

    ``reduce`` never synchronises.  Each call first checks the health words of the
    previous reduces that have already completed on the GPU and raises the reference's
    ``ValueError`` ("gradient vector contains NaN or Inf", core.py:157-158) for a rank
    whose gradient held NaN/Inf, or ``RuntimeError`` if the cross-rank exchange timed out
    (``timeout_s``, default 300 s; the output of such a step is all NaN, never a silently
    incomplete average).  ``check()`` waits for every outstanding reduce and raises the same.
    """

    def __init__(self, dim: int, rows: int = DEFAULT_ROWS, cols: int | None = None, seed: int = 0,
                 num_blocks: int | None = None, size_ratio: float = DEFAULT_SIZE_RATIO,
                 alpha: float | None = None, group=None, world: int | None = None, rank: int | None = None,
                 timeout_s: float = 0.0, exchange_grid: int = 0):
        import torch.distributed as dist

        if cols is None:
            if alpha is None:
                raise ValueError("give cols, or alpha (expected non-zero fraction) to size the sketch")
            cols = sketch_cols(size_ratio, alpha, dim, rows)
        self.dim, self.rows, self.cols, self.seed = int(dim), int(rows), int(cols), int(seed)
        self.num_blocks = int(num_blocks or dim)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.plan = Plan(self.dim, self.num_blocks, self.rows, self.cols, self.seed)
        if world is None:
            world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if world > 1 else 0
        self.world, self.rank = int(world), int(rank)
        uid = (ctypes.c_uint8 * 128)()
        mode = S2_COMM_IPC
        if self.world > 1:
            ctypes.memmove(uid, broadcast_unique_id(self.rank, group), 128)
            import os

            if os.environ.get("S2_AGG") == "nccl":  # north-star literal: NCCL all-reduce + all-gather + OR
                mode = S2_COMM_NCCL
        check(lib.s2_comm_set_options(self.plan.handle, int(exchange_grid), float(timeout_s)), "comm options")
        check(lib.s2_comm_init_mode(self.plan.handle, self.world, self.rank, uid, mode), "comm init")
        check(lib.s2_comm_check(self.plan.handle, stream_ptr()), "comm check")
        self._status = _StatusRing(self.plan.handle, self.device)

    def reduce(self, g: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Averaged gradient estimate: median-of-rows sketch query ÷ world at every union-bitmap
        coordinate, 0 elsewhere (sparse_decompress of sparse_merge of every rank's sparse_compress)."""
        if g.numel() != self.dim:
            raise ValueError(f"dimension mismatch: mask dim {self.dim}, vector {g.numel()}")
        self._status.poll()
        if not (g.is_cuda and g.dtype == torch.float32 and g.is_contiguous() and g.data_ptr() % 16 == 0):
            g = as_gradient(g, self.device)
        if out is None:
            out = torch.empty(self.dim, dtype=torch.float32, device=self.device)
        st = stream if stream is not None else torch.cuda.current_stream()
        k = self._status.arm()
        check(lib.s2_reduce(self.plan.handle, ptr(g), ptr(out), None, stream_ptr(st)), "reduce")
        self._status.launched(k, st)
        return out

    def reduce_many(self, gs, outs=None, stream=None):
        """``[reduce(g) for g in gs]`` as one pipelined batch (``s2_reduce_many``): with W > 1 the
        compress of step k+1 runs while step k's NVLink exchange is in flight.  Same outputs."""
        gs = list(gs)
        for g in gs:
            if g.numel() != self.dim:
                raise ValueError(f"dimension mismatch: mask dim {self.dim}, vector {g.numel()}")
        self._status.poll()
        gs = [g if (g.is_cuda and g.dtype == torch.float32 and g.is_contiguous() and g.data_ptr() % 16 == 0)
              else as_gradient(g, self.device) for g in gs]
        if outs is None:
            outs = [torch.empty(self.dim, dtype=torch.float32, device=self.device) for _ in gs]
        st = stream if stream is not None else torch.cuda.current_stream()
        gp = (ctypes.c_void_p * len(gs))(*[g.data_ptr() for g in gs])
        op = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        k = self._status.arm()
        check(lib.s2_reduce_many(self.plan.handle, gp, op, len(gs), stream_ptr(st)), "reduce_many")
        self._status.launched(k, st)
        return outs

    def check(self) -> None:
        """Wait for every outstanding reduce and raise for NaN/Inf or an exchange timeout."""
        self._status.poll(wait=True)

    def counters(self) -> list[int]:
        """Counters of the last reduce (synchronises the current stream): [nnz, nonfinite, selected, 0]."""
        host = (ctypes.c_uint64 * S2_NUM_COUNTERS)()
        check(lib.s2_read_counters(self.plan.handle, host, stream_ptr()), "counters")
        return [int(v) for v in host]

    def check_finite(self) -> None:
        """Raise the reference's ValueError if the last reduced gradient held NaN/Inf (syncs)."""
        if self.counters()[S2_CNT_NONFINITE]:
            raise ValueError("gradient vector contains NaN or Inf")

    def last_nnz(self) -> int:
        return self.counters()[S2_CNT_NNZ]

    def check_exchange(self) -> None:
        """Raise if a cross-rank barrier of the peer-memory exchange timed out (a rank died or the
        ranks' reduce sequences diverged); synchronises the device."""
        torch.cuda.synchronize(self.device)
        if lib.s2_p2p_error(self.plan.handle):
            raise RuntimeError("S2 exchange: a cross-rank barrier timed out")


class HostPipeline:
    """Reduce gradients that live in (pinned) host memory, overlapping PCIe with the GPU.

    ``submit(g_host, out_host)`` enqueues H2D of the gradient on a copy-in stream,
    the reduce on the compute stream and D2H of the result on a copy-out stream,
    with double-buffered device staging, so step i's reduce overlaps step i+1's
    H2D and step i-1's D2H (PCIe is full duplex).  It returns a CUDA event that
    completes when ``out_host`` holds the result; ``drain()`` waits for all.
    """

    def __init__(self, reducer: S2Reducer, depth: int = 2):
        self.r = reducer
        dev = reducer.device
        self.depth = depth
        self.s_in = torch.cuda.Stream(device=dev)
        self.s_comp = torch.cuda.Stream(device=dev)
        self.s_out = torch.cuda.Stream(device=dev)
        self.g = [torch.empty(reducer.dim, dtype=torch.float32, device=dev) for _ in range(depth)]
        self.o = [torch.empty(reducer.dim, dtype=torch.float32, device=dev) for _ in range(depth)]
        self.comp_done = [None] * depth  # reduce i finished reading g[i%depth] / writing o[i%depth]
        self.out_done = [None] * depth   # D2H of o[i%depth] finished
        self.i = 0

    def submit(self, g_host: torch.Tensor, out_host: torch.Tensor) -> torch.cuda.Event:
        k = self.i % self.depth
        self.i += 1
        with torch.cuda.stream(self.s_in):
            if self.comp_done[k] is not None:
                self.s_in.wait_event(self.comp_done[k])  # g[k] free again
            self.g[k].copy_(g_host, non_blocking=True)
            in_done = torch.cuda.Event()
            in_done.record(self.s_in)
        with torch.cuda.stream(self.s_comp):
            self.s_comp.wait_event(in_done)
            if self.out_done[k] is not None:
                self.s_comp.wait_event(self.out_done[k])  # o[k] drained to the host
            self.r.reduce(self.g[k], out=self.o[k], stream=self.s_comp)
            ev = torch.cuda.Event()
            ev.record(self.s_comp)
            self.comp_done[k] = ev
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(ev)
            out_host.copy_(self.o[k], non_blocking=True)
            od = torch.cuda.Event()
            od.record(self.s_out)
            self.out_done[k] = od
        return od

    def drain(self) -> None:
        for e in self.out_done:
            if e is not None:
                e.synchronize()


class GraphedReduce:
    """CUDA-graph replay of ``S2Reducer.reduce`` on static buffers (no per-step launch cost).

    The plan rotates its buffers with period 4 (sketch tables / counters over 4 slots, bitmaps
    over 2, s2_reduce), so four graphs are captured — one per slot — and ``__call__`` replays
    them in order.  Do not interleave direct ``reduce`` calls on the same reducer with replays
    (they advance the rotation too; a multiple of four of them is harmless).

        gr = GraphedReduce(reducer, g_static, out_static)
        g_static.copy_(grad); gr(); use(out_static)
    """

    def __init__(self, reducer: S2Reducer, g_static: torch.Tensor, out_static: torch.Tensor):
        self.r, self.g, self.out = reducer, g_static, out_static
        s = torch.cuda.Stream(device=reducer.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(4):  # warm-up: scratch allocated, every slot exercised
                reducer.reduce(g_static, out=out_static, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        reducer.check()
        self.graphs = []
        # each graph writes its health word into its own pinned slot (captured pointer)
        self.words = torch.zeros(4, dtype=torch.int32, pin_memory=True)
        for k in range(4):
            check(lib.s2_plan_set_status(reducer.plan.handle, ctypes.c_void_p(self.words.data_ptr() + 4 * k)),
                  "set status")
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                check(lib.s2_reduce(reducer.plan.handle, ptr(g_static), ptr(out_static), None, stream_ptr()),
                      "reduce")
            self.graphs.append(gph)
        check(lib.s2_plan_set_status(reducer.plan.handle, None), "set status")
        # capture advanced the rotation by four: back at the slot graph 0 was recorded in
        self.k = 0
        self.last = [None] * 4

    def __call__(self) -> torch.Tensor:
        k = self.k
        if self.last[k] is not None:  # this graph's previous replay must be checked before reuse
            self.last[k].synchronize()
            self._check(k)
        self.graphs[k].replay()
        ev = torch.cuda.Event()
        ev.record()
        self.last[k] = ev
        self.k = (k + 1) % 4
        return self.out

    def _check(self, k: int) -> None:
        st = int(self.words[k]) & 0xFFFFFFFF
        self.words[k] = 0  # the replay that wrote it has completed; re-arm for the next one
        if st & S2_STATUS_EXCHANGE:
            raise RuntimeError("S2 exchange: a cross-rank barrier timed out; the averaged gradient was set to NaN")
        if st & S2_STATUS_NONFINITE:
            raise ValueError("gradient vector contains NaN or Inf")

    def check(self) -> None:
        for k in range(4):
            if self.last[k] is not None:
                self.last[k].synchronize()
                self._check(k)
