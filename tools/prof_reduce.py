"""Short S2 reduce loop for ncu / compute-sanitizer captures (1 GPU).

    python tools/prof_reduce.py [--config resnet50] [--steps 6]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2110_02140_b200 import synthetic  # noqa: E402
import paper_2110_02140_b200 as s2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="resnet50")
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--block", type=int, default=0, help="num_blocks (0 = element bitmap)")
a = ap.parse_args()
cfg = CONFIGS[a.config]
d = cfg["dim"]
red = s2.S2Reducer(d, rows=cfg["rows"], cols=cfg["cols"], seed=0, num_blocks=a.block or cfg.get("num_blocks"))
gs = [synthetic.gradient(dict(dim=d, alpha=cfg["alpha"], rows=cfg.get("grid")), 0, base_seed=1234 + 1000 * k) for k in range(2)]
out = torch.empty(d, device="cuda")
for i in range(a.steps):
    red.reduce(gs[i % 2], out=out)
torch.cuda.synchronize()
red.check_finite()
print("ok", a.config, a.steps)
