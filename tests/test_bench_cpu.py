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


def test_kernel_floors():
    """bench.kernel_floors: HBM bytes at the peak vs REDs at the L2 RED rate (compress) and vs
    L1 -> crossbar requests (decode), whichever is larger, with the bound named."""
    sys.path.insert(0, ROOT)
    import bench

    d, rows, cols = 25_600_000, 3, 262_144
    wb = 4 * (-(-d // 32))
    f1 = bench.kernel_floors(d, rows, cols, wb, 256_000, 256_000, 6552.6)
    assert f1["compress"]["bound"] == "hbm" and f1["decode"]["bound"] == "hbm"
    assert abs(f1["compress"]["us"] - (4 * d + wb + 4 * rows * cols) / 6552.6e9 * 1e6) < 0.01
    assert f1["decode"]["requests"] == int(rows * 256_000 + (4 * d + 4 * rows * cols + wb) / 32)
    f8 = bench.kernel_floors(d, rows, cols, wb, 256_000, int(0.0773 * d), 6552.6)
    assert f8["decode"]["bound"] == "l1-xbar requests" and f8["decode"]["us"] > f1["decode"]["us"]
    fb = bench.kernel_floors(110_000_000, 5, 1 << 20, 4 * (110_000_000 // 32), 5_500_000, 5_500_000, 6552.6)
    assert fb["compress"]["bound"] == "l2 red"
    assert abs(fb["compress"]["us"] - 5 * 5_500_000 / bench.L2_RED_PER_S * 1e6) < 0.01
