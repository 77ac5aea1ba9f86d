"""Cross-GPU barrier latency sweep (experiment).  torchrun --nproc-per-node N tools/barrier_bench.py"""
import ctypes
import json
import os

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libbarrier.so"))
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
G = torch.cuda.get_device_properties(0).multi_processor_count
res = {}
for mode in (0, 1, 2, 3):
    for grid in (1, G):
        lib.bb_alloc.restype = ctypes.c_void_p
        fptr = lib.bb_alloc(ctypes.c_size_t(world * G * 4))  # own cudaMalloc: IPC handles map whole allocations
        h = (ctypes.c_uint8 * 64)()
        assert lib.bb_ipc_handle(ctypes.c_void_p(fptr), h) == 0
        hs = [None] * world
        dist.all_gather_object(hs, bytes(h))
        ptrs = (ctypes.c_void_p * world)()
        for q in range(world):
            if q == rank:
                ptrs[q] = fptr
            else:
                p = ctypes.c_void_p()
                assert lib.bb_ipc_open(hs[q], ctypes.byref(p)) == 0
                ptrs[q] = p
        out = torch.zeros(G, dtype=torch.int64, device="cuda")
        dist.barrier()
        rc = lib.bb_run(ptrs, world, rank, 200, mode, grid, 256, ctypes.c_void_p(out.data_ptr()))
        assert rc == 0, rc
        ns = out[:grid].cpu().numpy()
        res[f"mode{mode} grid{grid}"] = int(np.median(ns))
        dist.barrier()
if rank == 0:
    print(json.dumps({"world": world, "ns_per_barrier": res}))
dist.destroy_process_group()
