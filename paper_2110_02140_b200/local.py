"""W virtual ranks of the S2 reduce on ONE GPU — the single-GPU multi-rank harness.

Every rank gets its own plan and exchange arena (``S2_COMM_EXTERNAL``: no NCCL) and runs
``s2_reduce`` on its own CUDA stream, so the product's peer-memory exchange kernels
(``k_p2p_oneshot`` / ``k_p2p_aggregate``, csrc/s2_p2p.cu) execute exactly as on W GPUs —
the same arena layout, cross-rank flag barriers and rank-ordered sums — with the "peer"
arenas in the same device memory.  This lets a one-GPU box check the W = 2..8 exchange
against the oracle (sparse.py:174-196) and proxy the W = 8 union density for the decode.

The exchange grids of all W ranks must be co-resident (a CTA waits for the same CTA
index of the other ranks): each rank's exchange kernel gets ``exchange_grid`` CTAs of
1024 threads (one SM each), default SMs // (2W), so W x G SMs at most spin while the
rest of the GPU runs the ranks' compress and decode kernels.  The ranks' streams (two per
rank under ``reduce_many``) must not share CUDA hardware work queues, or a spinning exchange
can queue in front of work another rank waits for: set ``CUDA_DEVICE_MAX_CONNECTIONS`` >= 2W + 2
before CUDA initialises (tests/conftest.py sets 32).
"""

from __future__ import annotations

import ctypes
import os
import warnings

import torch

from ._lib import S2_COMM_EXTERNAL, check, lib, ptr
from .sketch import Plan


class LocalGroup:
    def __init__(self, world: int, dim: int, rows: int, cols: int, seed: int = 0, num_blocks: int | None = None,
                 exchange_grid: int = 0, timeout_s: float = 20.0):
        if not 2 <= world <= 8:
            raise ValueError("world must be in [2, 8]")
        conns = int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8"))
        if conns < 2 * world + 2:
            warnings.warn(f"CUDA_DEVICE_MAX_CONNECTIONS={conns} < {2 * world + 2}: the {world} ranks' streams share "
                          "hardware queues and a pipelined exchange may time out (see module docstring)")
        self.world, self.dim = int(world), int(dim)
        dev = torch.device("cuda", torch.cuda.current_device())
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self.grid = int(exchange_grid) or max(1, sms // (2 * world))
        self.plans = [Plan(dim, num_blocks or dim, rows, cols, seed) for _ in range(world)]
        digests = {int(lib.s2_plan_digest(p.handle)) for p in self.plans}
        if len(digests) != 1:  # sparse.py:179-187, checked on the host in EXTERNAL mode
            raise ValueError("incompatible payloads: field 'sketch_params' differs")
        for r, p in enumerate(self.plans):
            check(lib.s2_comm_set_options(p.handle, self.grid, float(timeout_s)), "comm options")
            check(lib.s2_comm_init_mode(p.handle, world, r, None, S2_COMM_EXTERNAL), "comm init")
        nbytes = int(lib.s2_p2p_arena_bytes(self.plans[0].handle, world))
        if nbytes <= 0:
            raise RuntimeError("s2_p2p_arena_bytes failed")
        # one arena per rank; the caching allocator returns >= 512-byte aligned blocks
        self.arenas = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(world)]
        bases = (ctypes.c_uint64 * world)(*[a.data_ptr() for a in self.arenas])
        torch.cuda.synchronize()
        for p in self.plans:
            check(lib.s2_comm_attach(p.handle, bases, world), "comm attach")
        torch.cuda.synchronize()
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(world)]

    def reduce(self, grads, outs=None):
        """Rank r reduces grads[r] into outs[r] on its own stream; returns outs (every rank's
        averaged estimate, identical on all ranks).  Stream-ordered after the current stream."""
        if len(grads) != self.world:
            raise ValueError("need one gradient per rank")
        if outs is None:
            outs = [torch.empty(self.dim, dtype=torch.float32, device=g.device) for g in grads]
        cur = torch.cuda.current_stream()
        for r, (p, g, o, s) in enumerate(zip(self.plans, grads, outs, self.streams)):
            s.wait_stream(cur)
            check(lib.s2_reduce(p.handle, ptr(g), ptr(o), None, ctypes.c_void_p(s.cuda_stream)), f"reduce rank {r}")
        for g, o, s in zip(grads, outs, self.streams):
            cur.wait_stream(s)
            g.record_stream(s)
            o.record_stream(s)
        return outs

    def reduce_many(self, steps):
        """steps[k][r] = rank r's gradient of step k; every rank runs s2_reduce_many (the pipelined
        batch) on its own stream.  Returns outs[k][r]."""
        n = len(steps)
        outs = [[torch.empty(self.dim, dtype=torch.float32, device=g.device) for g in st] for st in steps]
        cur = torch.cuda.current_stream()
        for r, (p, s) in enumerate(zip(self.plans, self.streams)):
            s.wait_stream(cur)
            gp = (ctypes.c_void_p * n)(*[steps[k][r].data_ptr() for k in range(n)])
            op = (ctypes.c_void_p * n)(*[outs[k][r].data_ptr() for k in range(n)])
            check(lib.s2_reduce_many(p.handle, gp, op, n, ctypes.c_void_p(s.cuda_stream)), f"reduce_many rank {r}")
        for s in self.streams:
            cur.wait_stream(s)
        for k in range(n):
            for r, s in enumerate(self.streams):
                steps[k][r].record_stream(s)
                outs[k][r].record_stream(s)
        return outs

    def set_status(self, words: torch.Tensor) -> None:
        """words: int32[world] (device or pinned host); rank r's later reduces write their
        S2_STATUS_* bits into words[r]."""
        for r, p in enumerate(self.plans):
            check(lib.s2_plan_set_status(p.handle, ctypes.c_void_p(words.data_ptr() + 4 * r)), "set status")

    def errors(self) -> list[int]:
        """Sticky exchange-timeout word of every rank (synchronises)."""
        torch.cuda.synchronize()
        return [int(lib.s2_p2p_error(p.handle)) for p in self.plans]
