"""Probe torch symmetric memory + NVLS multicast availability (torchrun, 2+ ranks)."""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
info = {"rank": rank}
try:
    info["backend"] = symm_mem.get_backend(torch.device("cuda", rank))
except Exception as e:  # noqa: BLE001
    info["backend_err"] = repr(e)
try:
    info["has_mc"] = bool(symm_mem._SymmetricMemory.has_multicast_support(symm_mem.DeviceType.CUDA, rank))
except Exception as e:  # noqa: BLE001
    info["has_mc_err"] = repr(e)
try:
    t = symm_mem.empty(1 << 20, dtype=torch.uint8, device=f"cuda:{rank}")
    h = symm_mem.rendezvous(t, dist.group.WORLD)
    info["buffer_ptrs"] = [hex(p) for p in h.buffer_ptrs]
    info["mc_ptr"] = hex(h.multicast_ptr) if hasattr(h, "multicast_ptr") else None
    info["t_ptr"] = hex(t.data_ptr())
    info["signal_pad_size"] = symm_mem.get_signal_pad_size()
    info["attrs"] = [a for a in dir(h) if not a.startswith("_")]
except Exception as e:  # noqa: BLE001
    info["rdv_err"] = repr(e)
print(info, flush=True)
dist.destroy_process_group()
