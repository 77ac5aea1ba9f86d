"""Training-loop caller: S2 sparse-sketch reduce as a torch DDP communication hook.

SURVEY.md §8(f) rank 2.  The reference drives its compressors through
``casq.ef_step`` (casq.py:315-332): ``g~ = lr*grad + e``, compress ``g~``,
``g^ = decompress(merge(payloads))`` and carry ``e' = g~ - g^`` — in a multi-worker
loop the residual is taken against the merged estimate.  This hook does exactly that
per DDP gradient bucket (``lr`` folded in by the optimizer, so the hook uses 1) through
``ef.ef_reduce``:

    model = DDP(model)
    model.register_comm_hook(S2HookState(size_ratio=0.5, alpha=0.01), s2_comm_hook)

The bucket's flat gradient is reduced by ``S2Reducer`` (compress -> NVLink exchange ->
median decode, averaged over ranks) on the current stream; DDP receives the estimate.
Errors surface without a host sync: ``S2Reducer.reduce`` raises the reference's
``ValueError`` ("gradient vector contains NaN or Inf", core.py:157-158) or a
``RuntimeError`` (exchange timeout) for an earlier step as soon as that step has
completed on the GPU; ``S2HookState.check()`` waits for all of them (e.g. once per epoch).

Error-feedback residuals are keyed by the identity of the bucket's parameters, not by
``bucket.index()``: DDP rebuilds its buckets after the first iteration and indices are
not stable (torch GradBucket docs).  When a bucket's parameter set changes, the residuals
of the buckets it replaces are dropped.  Error feedback is opt-in
(``error_feedback=True``): with W > 1 the residual taken against the merged estimate is
non-zero wherever ANY rank had a non-zero, so the compressed vector densifies step by
step and the sketch (sized for alpha) saturates unless alpha/size_ratio account for it.
"""

import torch
import torch.distributed as dist

from .ef import ErrorState, ef_reduce
from .reducer import S2Reducer
from .sparse import DEFAULT_ROWS, DEFAULT_SIZE_RATIO, sketch_cols


class S2HookState:
    """Per-process hook state: one S2Reducer (plan + exchange arena) per bucket size and an
    error-feedback residual per bucket parameter set."""

    def __init__(self, process_group=None, rows: int = DEFAULT_ROWS, size_ratio: float = DEFAULT_SIZE_RATIO,
                 alpha: float = 0.01, seed: int = 0, error_feedback: bool = False, timeout_s: float = 0.0):
        self.group = process_group
        self.rows, self.size_ratio, self.alpha, self.seed = rows, size_ratio, alpha, seed
        self.error_feedback = error_feedback
        self.timeout_s = timeout_s
        self.reducers = {}    # bucket numel -> S2Reducer
        self.residuals = {}   # tuple(id(param) ...) -> ErrorState
        self._owner = {}      # id(param) -> residual key holding it

    def reducer(self, numel: int) -> S2Reducer:
        r = self.reducers.get(numel)
        if r is None:
            cols = sketch_cols(self.size_ratio, self.alpha, numel, self.rows)
            r = S2Reducer(numel, rows=self.rows, cols=cols, seed=self.seed, group=self.group,
                          timeout_s=self.timeout_s)
            self.reducers[numel] = r
        return r

    def residual(self, key: tuple, numel: int, device) -> ErrorState:
        st = self.residuals.get(key)
        if st is None or st.e.numel() != numel:
            for pid in key:  # the bucket layout changed: drop the residuals of the buckets it replaces
                old = self._owner.get(pid)
                if old is not None and old != key:
                    self.residuals.pop(old, None)
                self._owner[pid] = key
            st = ErrorState.zeros(numel, device=device)
            self.residuals[key] = st
        return st

    def check(self) -> None:
        """Wait for every outstanding reduce; raise for NaN/Inf or an exchange timeout."""
        for r in self.reducers.values():
            r.check()


def s2_comm_hook(state: S2HookState, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    g = bucket.buffer()
    flat = g.reshape(-1)
    if flat.dtype != torch.float32:
        raise TypeError("s2_comm_hook reduces float32 gradients")
    red = state.reducer(flat.numel())
    if state.error_feedback:
        key = tuple(id(p) for p in bucket.parameters())
        st = state.residual(key, flat.numel(), flat.device)
        est, state.residuals[key] = ef_reduce(st, flat, 1.0, red)  # g~ = grad + e; e' = g~ - g^
    else:
        est = red.reduce(flat if flat.data_ptr() % 16 == 0 else flat.contiguous().clone())
    flat.copy_(est)
    fut = torch.futures.Future()
    fut.set_result(g)
    return fut
