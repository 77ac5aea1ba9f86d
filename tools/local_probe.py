"""Probe the single-GPU multi-rank harness for cross-stream co-scheduling failures: many fresh
LocalGroups (W = 2..4), short barrier timeout; counts reduces whose exchange timed out.
Run with and without CUDA_DEVICE_MAX_CONNECTIONS=32."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from oracle import s2_oracle as o  # noqa: E402
from paper_2110_02140_b200.local import LocalGroup  # noqa: E402

dim = 200_003
res = {"CUDA_DEVICE_MAX_CONNECTIONS": os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS")}
for W in (2, 3, 4):
    bad = 0
    tot = 0
    for trial in range(8):
        grp = LocalGroup(W, dim, 3, 4099, timeout_s=2.0)
        words = torch.full((W,), -1, dtype=torch.int32, device="cuda")
        grp.set_status(words)
        gt = [torch.from_numpy(o.synthetic_gradient(dim, 0.01, r, kind="int")).cuda() for r in range(W)]
        for _ in range(2):
            outs = grp.reduce(gt)
            torch.cuda.synchronize()
            tot += 1
            if any(int(x) != 0 for x in words.cpu()):
                bad += 1
        del grp
    res[f"W{W}"] = {"timed_out_reduces": bad, "reduces": tot}
print(json.dumps(res))
