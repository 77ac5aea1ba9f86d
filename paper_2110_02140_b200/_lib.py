"""ctypes binding of libs2.so (the C ABI in include/s2.h).

The library is built in-tree by ``paper_2110_02140_b200.build`` (or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing, importing this module raises, so no operation can silently run on
the CPU.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int8, c_int64, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("S2_LIB") or os.path.join(_HERE, "libs2.so")  # S2_LIB: A/B of two builds

S2_OK = 0
S2_EINVAL = 1
S2_ENONFINITE = 2
S2_ECUDA = 3
S2_ENCCL = 4
S2_EINCOMPAT = 5
S2_MAX_ROWS = 16
S2_CNT_NNZ = 0
S2_CNT_NONFINITE = 1
S2_CNT_SELECTED = 2
S2_NUM_COUNTERS = 4
S2_MASK_NONZERO = 0
S2_MASK_GIVEN = 1
S2_STATUS_NONFINITE = 1
S2_STATUS_EXCHANGE = 2
S2_COMM_IPC = 0
S2_COMM_NCCL = 1
S2_COMM_EXTERNAL = 2

# every symbol include/s2.h declares: name -> (restype, argtypes)
SIGNATURES = {
    "s2_last_error": (c_char_p, []),
    "s2_abi_version": (c_int, []),
    "s2_mix64": (c_uint64, [c_uint64]),
    "s2_derive_seed": (c_uint64, [POINTER(c_uint64), c_int]),
    "s2_row_seeds": (c_int, [c_uint64, c_int, POINTER(c_uint64)]),
    "s2_hash_host": (c_int, [c_uint64, POINTER(c_int64), c_int64, c_int64, POINTER(c_int64), POINTER(c_int8)]),
    "s2_plan_create": (c_int, [c_int64, c_int64, c_int, c_int64, c_uint64, c_int, POINTER(c_void_p)]),
    "s2_plan_destroy": (None, [c_void_p]),
    "s2_plan_bitmap_words": (c_int64, [c_void_p]),
    "s2_plan_block_size": (c_int64, [c_void_p]),
    "s2_compress": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "s2_decode": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "s2_sketch_insert": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "s2_sketch_query": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "s2_bitmap_or": (c_int, [c_int64, c_void_p, c_int, c_void_p, c_void_p]),
    "s2_table_sum": (c_int, [c_int64, c_void_p, c_int, c_void_p, c_void_p]),
    "s2_selected_count": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "s2_compact_scratch_bytes": (c_int64, [c_void_p]),
    "s2_block_topk_scratch_bytes": (c_int64, [c_void_p]),
    "s2_block_topk": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "s2_compact": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "s2_nccl_unique_id": (c_int, [c_void_p]),
    "s2_comm_set_options": (c_int, [c_void_p, c_int, ctypes.c_double]),
    "s2_comm_init": (c_int, [c_void_p, c_int, c_int, c_void_p]),
    "s2_comm_init_mode": (c_int, [c_void_p, c_int, c_int, c_void_p, c_int]),
    "s2_p2p_arena_bytes": (c_int64, [c_void_p, c_int]),
    "s2_comm_attach": (c_int, [c_void_p, POINTER(c_uint64), c_int]),
    "s2_plan_digest": (c_uint64, [c_void_p]),
    "s2_plan_set_status": (c_int, [c_void_p, c_void_p]),
    "s2_comm_check": (c_int, [c_void_p, c_void_p]),
    "s2_aggregate": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "s2_reduce": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "s2_reduce_many": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "s2_plan_world": (c_int, [c_void_p]),
    "s2_last_counters": (c_void_p, [c_void_p]),
    "s2_read_counters": (c_int, [c_void_p, c_void_p, c_void_p]),
    "s2_plan_set_timing_events": (c_int, [c_void_p, c_void_p, c_int]),
    "s2_p2p_trace": (c_int, [c_void_p, c_void_p, c_int64]),
    "s2_p2p_error": (c_int, [c_void_p]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2110_02140_b200/build.py` "
            "(there is no CPU fallback for the S2 path)"
        )
    # make sure torch's libnccl/libcudart are loaded first so libs2.so binds to the same copies
    import torch  # noqa: F401

    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class S2Error(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    """Map a status code to the reference's exception types (ValueError for argument errors)."""
    if rc == S2_OK:
        return
    msg = lib.s2_last_error().decode(errors="replace")
    if rc in (S2_EINVAL, S2_ENONFINITE, S2_EINCOMPAT):
        raise ValueError(msg)
    raise S2Error(f"{what}: {msg}" if what else msg)


def ptr(t) -> c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    return c_void_p(0 if t is None else t.data_ptr())


def stream_ptr(stream=None) -> c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return c_void_p(s.cuda_stream)


__all__ = ["lib", "check", "ptr", "stream_ptr", "S2Error", "LIB_PATH", "SIGNATURES"]
_ = (c_float,)
