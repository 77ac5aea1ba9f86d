"""GPT-2-medium sweep of BASELINE.json configs[4]: sparsity 90-99.9 % x sketch width 2^16..2^22.

    python tools/sweep_gpt2.py [--gpus N] > sweep.jsonl   (N > 1 launches torchrun per point)
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=1)
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
for alpha in (0.10, 0.05, 0.01, 0.001):
    for cols in (1 << 16, 1 << 18, 1 << 20, 1 << 22):
        base = ["bench.py", "--config", "gpt2m_90", "--alpha", str(alpha), "--cols", str(cols),
                "--steps", str(a.steps), "--no-cpu-baseline", "--gpus", str(a.gpus)]
        if a.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
                   "--master-addr", "127.0.0.1", "--master-port", str(29800 + (cols.bit_length() % 50))] + base
        else:
            cmd = [sys.executable] + base
        r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
        lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
        if not lines:
            print(json.dumps({"alpha": alpha, "cols": cols, "error": r.stderr[-400:]}), flush=True)
            continue
        d = json.loads(lines[-1])
        print(json.dumps({"alpha": alpha, "cols": cols, "gpus": a.gpus, "ms": d["ms_per_step"],
                          "latency_ms": d.get("latency_ms_per_reduce"), "GBps_per_gpu": d["value"],
                          "GBps_job": d.get("job_GBps"), "phases": d["phases"]}), flush=True)
