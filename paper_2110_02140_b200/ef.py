"""Error feedback around the S2 compressor — the reference's training-loop caller.

Mirrors ``ErrorState`` / ``ef_step`` (/root/reference/pkg/src/sketchgrad/casq.py:303-332) on
CUDA tensors: ``g~ = lr * grad + e``, compress ``g~``, ``g^ = decompress(merge([payload]))``,
``e' = g~ - g^``.  In a multi-worker loop the residual is taken against the merged estimate
(casq.py:323-324), which is what ``ef_reduce`` does with the distributed ``S2Reducer``.
The residual is kept in float32 on the GPU (the reference keeps float64 on the host); on
integer-valued (or dyadic) inputs the two are identical.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .core import as_gradient


@dataclass
class ErrorState:
    """Per-worker error-compensation vector (starts at zero), casq.py:303-312."""

    e: torch.Tensor
    worker_id: int = 0

    @classmethod
    def zeros(cls, dim: int, worker_id: int = 0, device=None) -> "ErrorState":
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        return cls(torch.zeros(int(dim), dtype=torch.float32, device=dev), worker_id)


def _tilde(state: ErrorState, grad, lr: float) -> torch.Tensor:
    grad = as_gradient(grad, state.e.device)
    if grad.numel() != state.e.numel():
        raise ValueError("error state dimension does not match gradient")  # casq.py:325-326
    if lr <= 0:
        raise ValueError("learning rate must be positive")  # casq.py:327-328
    return grad * lr + state.e if lr != 1.0 else grad + state.e  # g~ = lr*grad + e (casq.py:329)


def ef_step(state: ErrorState, grad, lr: float, compressor):
    """One local error-feedback step through ``compressor`` (casq.py:315-332).
    Returns (payload, estimate, new state)."""
    g_tilde = _tilde(state, grad, lr)
    payload = compressor.compress(g_tilde)
    g_hat = compressor.decompress(compressor.merge([payload]))
    return payload, g_hat, ErrorState(g_tilde - g_hat, state.worker_id)


def ef_reduce(state: ErrorState, grad, lr: float, reducer):
    """The multi-worker form: the residual is taken against the MERGED estimate (the averaged
    reduce of every rank's g~, casq.py:323-324).  Returns (estimate, new state)."""
    g_tilde = _tilde(state, grad, lr)
    g_hat = reducer.reduce(g_tilde)
    return g_hat, ErrorState(g_tilde - g_hat, state.worker_id)
