import os
import sys

# The single-GPU multi-rank harness (tests/test_local_ranks.py) runs W ranks x 2 streams
# (s2_reduce_many's exchange stream) in one process.  With CUDA's default 8 hardware work queues,
# streams share queues and a spinning exchange kernel can sit in front of the compress another
# rank's exchange waits for (false dependency -> barrier timeout).  Must be set before the CUDA
# context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def _ensure_built():
    """libs2.so is git-ignored: build it in-tree (nvcc cross-compiles sm_100a without a GPU)
    when a fresh checkout runs the tests before __graft_entry__.build()."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("s2_build", os.path.join(ROOT, "paper_2110_02140_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build(force=False, verbose=False)


_ensure_built()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
