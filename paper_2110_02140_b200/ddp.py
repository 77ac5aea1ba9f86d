"""Training-loop caller: S2 sparse-sketch reduce as a torch DDP communication hook.

SURVEY.md §8(f) rank 2.  The reference drives its compressors through
``casq.ef_step`` (casq.py:315-332): ``g~ = lr*grad + e``, compress ``g~``,
``g^ = decompress(merge(payloads))`` and carry ``e' = g~ - g^`` — in a multi-worker
loop the residual is taken against the merged estimate.  This hook does exactly that
per DDP gradient bucket (``lr`` folded in by the optimizer, so the hook uses 1):

    model = DDP(model)
    model.register_comm_hook(S2HookState(size_ratio=0.5, alpha=0.01), s2_comm_hook)

The bucket's flat gradient is reduced by ``S2Reducer`` (compress -> NVLink exchange ->
median decode, averaged over ranks) on the current stream; DDP receives the estimate.

Error feedback is opt-in (``error_feedback=True``): with W > 1 the residual taken
against the merged estimate is non-zero wherever ANY rank had a non-zero, so the
compressed vector densifies step by step and the sketch (sized for alpha) saturates
unless alpha/size_ratio account for it (measured in tools/ddp_check.py).
"""

import torch
import torch.distributed as dist

from .reducer import S2Reducer
from .sparse import DEFAULT_ROWS, DEFAULT_SIZE_RATIO, sketch_cols


class S2HookState:
    """Per-process hook state: one S2Reducer (plan + exchange arena) per bucket size and an
    error-feedback residual per bucket index."""

    def __init__(self, process_group=None, rows: int = DEFAULT_ROWS, size_ratio: float = DEFAULT_SIZE_RATIO,
                 alpha: float = 0.01, seed: int = 0, error_feedback: bool = False):
        self.group = process_group
        self.rows, self.size_ratio, self.alpha, self.seed = rows, size_ratio, alpha, seed
        self.error_feedback = error_feedback
        self.reducers = {}   # bucket numel -> S2Reducer
        self.residuals = {}  # bucket index -> error-feedback residual

    def reducer(self, numel: int) -> S2Reducer:
        r = self.reducers.get(numel)
        if r is None:
            cols = sketch_cols(self.size_ratio, self.alpha, numel, self.rows)
            r = S2Reducer(numel, rows=self.rows, cols=cols, seed=self.seed, group=self.group)
            self.reducers[numel] = r
        return r


def s2_comm_hook(state: S2HookState, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    g = bucket.buffer()
    flat = g.reshape(-1)
    if flat.dtype != torch.float32:
        raise TypeError("s2_comm_hook reduces float32 gradients")
    red = state.reducer(flat.numel())
    if state.error_feedback:
        e = state.residuals.get(bucket.index())
        g_tilde = flat if e is None else flat + e  # ef_step: g~ = grad + e (casq.py:329)
    else:
        g_tilde = flat
    if not g_tilde.is_contiguous() or g_tilde.data_ptr() % 16:
        g_tilde = g_tilde.contiguous().clone()
    est = red.reduce(g_tilde)  # averaged estimate over ranks
    if state.error_feedback:
        state.residuals[bucket.index()] = g_tilde - est  # e' = g~ - g^ (casq.py:331)
    flat.copy_(est)
    fut = torch.futures.Future()
    fut.set_result(g)
    return fut
