"""The training-loop caller: error feedback around the S2 compressor
(casq.py:303-332) and the DDP comm hook, checked against the oracle on one GPU."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from oracle import s2_oracle as o

pytestmark = pytest.mark.gpu


def test_ef_step_matches_oracle_loop():
    """Three ef_step iterations (lr = 0.5) through SparseSketchCompressor(mask="nonzero") against
    the oracle's ef loop: g~ = lr*g + e, g^ = decompress(merge([compress(g~)])), e' = g~ - g^.
    Integer gradients and lr = 1/2 keep every value dyadic, so estimates and residuals are
    bit-exact although the GPU keeps the residual in float32 and the reference in float64."""
    import torch

    import paper_2110_02140_b200 as s2
    from paper_2110_02140_b200.ef import ErrorState, ef_step

    d = 200_003
    comp = s2.SparseSketchCompressor(d, d, 4000, mask="nonzero", seed=11)
    st = ErrorState.zeros(d)
    e_ref = np.zeros(d)
    for step in range(3):
        g = o.synthetic_gradient(d, 0.01, step, kind="int")
        pay, est, st = ef_step(st, torch.from_numpy(g).cuda(), 0.5, comp)
        g_t = 0.5 * g.astype(np.float64) + e_ref  # casq.py:329
        p = o.compress(g_t, g_t != 0, comp.rows, comp.cols, 11)
        ref = o.decompress(o.merge([p]))  # casq.py:330
        e_ref = g_t - ref  # casq.py:331
        assert np.array_equal(est.cpu().numpy(), ref.astype(np.float32)), step
        assert np.array_equal(st.e.cpu().numpy(), e_ref.astype(np.float32)), step
        assert pay.nnz == int((g_t != 0).sum())
    assert np.abs(e_ref).sum() > 0  # the residual is really carried
    with pytest.raises(ValueError, match="learning rate must be positive"):
        ef_step(st, torch.zeros(d, device="cuda"), 0.0, comp)
    with pytest.raises(ValueError, match="error state dimension does not match gradient"):
        ef_step(st, torch.zeros(d + 1, device="cuda"), 1.0, comp)


def test_ddp_hook_error_feedback_world1():
    """DDP with several buckets and error feedback (tests/ddp_ef_world1.py): estimates within the
    fp32 tolerance of the oracle, residual bookkeeping exact, residuals keyed by parameters."""
    env = dict(os.environ, S2_TEST_PORT="29613", PYTHONPATH=ROOT)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "ddp_ef_world1.py")], capture_output=True,
                       text=True, timeout=600, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    rep = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert rep["ok"], rep
