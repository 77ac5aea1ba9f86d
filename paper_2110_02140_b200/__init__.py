"""B200-native S2 Reducer sparse-sketch gradient reduce (arXiv 2110.02140).

Public API mirrors /root/reference/pkg/src/sketchgrad/sparse.py on CUDA
tensors; all compute runs in the sm_100a kernels of ``libs2.so``.
"""

from .core import BlockPartition, derive_seed, hash_buckets, hash_signs, mix64, row_seeds  # noqa: F401
from .reducer import S2Reducer  # noqa: F401
from .sketch import CountSketchTable, merge  # noqa: F401
from .ef import ErrorState, ef_reduce, ef_step  # noqa: F401
from .sparse import (DEFAULT_ROWS, DEFAULT_SIZE_RATIO, BlockMask, CommCost, SparsePayload,  # noqa: F401
                     SparseSketchCompressor, block_topk, compacted_values, mask_from_bytes, nonzero_mask,
                     sketch_cols, sparse_comm_bits, sparse_compress, sparse_decompress, sparse_merge,
                     sparse_payload_from_bytes, sparsify, topk_delta_check)

__all__ = [
    "BlockPartition", "BlockMask", "SparsePayload", "SparseSketchCompressor", "CountSketchTable", "S2Reducer",
    "sparse_compress", "sparse_merge", "sparse_decompress", "sparse_payload_from_bytes", "mask_from_bytes",
    "block_topk", "sketch_cols", "nonzero_mask", "compacted_values", "merge", "mix64", "derive_seed",
    "row_seeds", "hash_buckets", "hash_signs", "CommCost", "sparse_comm_bits", "sparsify", "topk_delta_check",
    "ErrorState", "ef_step", "ef_reduce",
]
