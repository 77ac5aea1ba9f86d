"""CPU: bench.py's reference arm (oracle port on the host cores) prints the contract's JSON
line, at N = 1 and under torchrun at N = 2 (rank 0 alone prints; the other rank exits 0)."""

import json
import os
import subprocess
import sys

from conftest import ROOT

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _check(out, n):
    lines = [x for x in out.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == n and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("oracle1m")


def test_reference_arm_n1():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "oracle1m", "--steps", "3",
                        "--warmup", "1", "--ref-budget", "2"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    _check(r.stdout, 1)


def test_reference_arm_torchrun_n2():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29651", "bench.py", "--gpus", "2",
                        "--impl", "reference", "--config", "oracle1m", "--steps", "3", "--warmup", "1",
                        "--ref-budget", "2"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    _check(r.stdout, 2)


def test_cpu_baseline_reports_as_shipped():
    """The ours-arm cpu_baseline carries the oracle port on all cores and the as-shipped call
    structure (single core, Python slice loops) at configs[0]."""
    sys.path.insert(0, ROOT)
    import bench

    cb = bench.cpu_baseline(bench.CONFIGS["oracle1m"], budget_s=1.0)
    assert cb["kind"] == "port" and cb["value"] > 0 and cb["cores"] >= 1
    a = cb["as_shipped"]
    assert a["kind"] == "port-as-shipped" and a["cores"] == 1 and 0 < a["value"] < cb["value"]
