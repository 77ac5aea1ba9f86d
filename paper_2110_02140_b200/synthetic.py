"""Synthetic sparse gradients for benchmarks (SURVEY.md §8(d) "Synthetic inputs").

``numpy_gradient`` follows the exact recipe the oracle/test fixtures use
(``default_rng(1234 + rank).choice(d, nnz, replace=False)`` positions, standard-normal
fp32 values) so CPU and GPU see identical bytes; ``cuda_gradient`` draws the same
shape of input directly on the GPU (fast for the 110M-355M configs).  ``rows`` builds
the embedding-style row-sparse gradient of the LSTM config: a V x H matrix with a
fraction of full non-zero rows.
"""

from __future__ import annotations

import numpy as np


def numpy_gradient(dim: int, alpha: float, rank: int = 0, base_seed: int = 1234) -> np.ndarray:
    rng = np.random.default_rng(base_seed + rank)
    nnz = int(round(alpha * dim))
    pos = rng.choice(dim, nnz, replace=False)
    vals = rng.standard_normal(nnz).astype(np.float32)
    vals[vals == 0] = 1.0
    g = np.zeros(dim, dtype=np.float32)
    g[pos] = vals
    return g


def zipf_weights(V: int, s: float) -> np.ndarray:
    """Row-draw probabilities p_i ~ 1/(i+1)^s: a vocabulary sorted by frequency, so ranks' rows overlap."""
    w = 1.0 / np.arange(1, V + 1, dtype=np.float64) ** s
    return w / w.sum()


def cuda_gradient(dim: int, alpha: float, rank: int = 0, base_seed: int = 1234, rows: tuple | None = None,
                  device="cuda", zipf: float | None = None):
    """fp32 CUDA gradient with round(alpha*dim) non-zeros at distinct random positions, or (rows=(V, H))
    round(alpha*V) full non-zero rows of a V x H row-major matrix (uniform rows, or Zipf(zipf) rows)."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(base_seed + 7919 * rank)
    g = torch.zeros(dim, dtype=torch.float32, device=device)
    if rows is not None:
        V, H = rows
        k = max(1, int(round(alpha * V)))
        if zipf:
            w = torch.from_numpy(zipf_weights(V, zipf)).to(device)
            r = torch.multinomial(w, k, replacement=False, generator=gen)
        else:
            r = torch.randperm(V, generator=gen, device=device)[:k]
        idx = (r[:, None] * H + torch.arange(H, device=device)[None, :]).reshape(-1)
    else:
        k = int(round(alpha * dim))
        idx = torch.randperm(dim, generator=gen, device=device)[:k]
    v = torch.randn(idx.numel(), generator=gen, device=device)
    v[v == 0] = 1.0
    g[idx] = v
    return g


def gradient(cfg: dict, rank: int = 0, base_seed: int = 1234, device="cuda"):
    """Bench input for a config dict (dim, alpha, optional rows=(V, H)); numpy recipe up to 50M elements."""
    import torch

    if cfg.get("rows") is None and cfg["dim"] <= 50_000_000:
        return torch.from_numpy(numpy_gradient(cfg["dim"], cfg["alpha"], rank, base_seed)).to(device)
    return cuda_gradient(cfg["dim"], cfg["alpha"], rank, base_seed, rows=cfg.get("rows"), device=device,
                         zipf=cfg.get("zipf"))
