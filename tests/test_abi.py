"""CPU: the C-ABI library loads, exports every symbol include/s2.h declares, and its host-side
logic (hash family, plan validation, error mapping) matches the golden vectors.  No device
compute is issued here."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "s2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(s2_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2110_02140_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares a signature for each one
    assert sorted(_lib.SIGNATURES) == syms


def test_abi_version_and_errors():
    from paper_2110_02140_b200._lib import check, lib

    assert lib.s2_abi_version() == 2
    h = ctypes.c_void_p()
    with pytest.raises(ValueError, match="rows and cols must be >= 1"):
        check(lib.s2_plan_create(10, 10, 0, 4, 0, 0, ctypes.byref(h)))
    with pytest.raises(ValueError, match=r"num_blocks must be in \[1, dim=10\]"):
        check(lib.s2_plan_create(10, 11, 3, 4, 0, 0, ctypes.byref(h)))
    with pytest.raises(ValueError, match="dim must be >= 1"):
        check(lib.s2_plan_create(0, 1, 3, 4, 0, 0, ctypes.byref(h)))
    with pytest.raises(ValueError, match="cols must be < 2"):
        check(lib.s2_plan_create(10, 10, 3, 2**32, 0, 0, ctypes.byref(h)))
    check(lib.s2_plan_create(10007, 1000, 3, 211, 0, 0, ctypes.byref(h)))
    assert lib.s2_plan_block_size(h) == 11 and lib.s2_plan_bitmap_words(h) == 32
    assert lib.s2_plan_world(h) == 1
    lib.s2_plan_destroy(h)


def test_host_hash_matches_golden():
    """The bucket/sign code the kernels inline (s2_common.cuh), compiled for the host, against the
    reference's own hash_buckets/hash_signs — incl. non-power-of-two cols via the magic divide."""
    import paper_2110_02140_b200 as s2

    z = np.load(os.path.join(GOLDEN, "hash_kat.npz"))
    for si, s in enumerate(z["derive_seeds_in"]):
        for jj, j in enumerate(z["derive_j"]):
            assert s2.derive_seed(int(s), int(j)) == int(z["derive_out"][si, jj])
    assert np.array_equal(s2.mix64(z["mix_in"]), z["mix_out"])
    for si, s in enumerate(z["row_seeds"]):
        assert np.array_equal(s2.hash_signs(int(s), z["idx"]), z["signs"][si])
        for ci, c in enumerate(z["cols"]):
            got = s2.hash_buckets(int(s), z["idx"], int(c))
            assert np.array_equal(got, z["buckets"][si, ci].astype(np.int64)), (si, int(c))


def test_magic_divide_exhaustive_edges():
    """floor(x / c) via multiply-high must be exact for every 63-bit x; probe the worst cases:
    x near multiples of c and near 2^63 for many non-power-of-two c (vs Python big ints)."""
    import paper_2110_02140_b200 as s2
    from oracle import s2_oracle as o

    rng = np.random.default_rng(5)
    cols_list = [3, 5, 7, 1000, 1667, 8334, 1_000_000, 2**20 + 1, 2**31 - 1, 2**31 + 1, 2**32 - 1,
                 *rng.integers(2, 2**32 - 1, size=20).tolist()]
    idx = rng.integers(0, 2**32 - 1, size=3000)
    seed = o.row_seeds(7, 1)[0]
    for c in cols_list:
        c = int(c)
        if c & (c - 1) == 0:
            continue
        assert np.array_equal(s2.hash_buckets(seed, idx, c), o.hash_buckets(seed, idx, c)), c


def test_row_seeds():
    import paper_2110_02140_b200 as s2
    from oracle import s2_oracle as o

    for seed in (0, 1, 42, 2**64 - 1):
        assert s2.row_seeds(seed, 16) == o.row_seeds(seed, 16)


def test_partition_mirror():
    import paper_2110_02140_b200 as s2
    from oracle import s2_oracle as o

    p = s2.BlockPartition(10007, 1000)
    assert p.block_size == 11
    assert np.array_equal(p.sizes(), o.block_sizes(10007, 1000))
    assert p.sizes().sum() == 10007 and (p.sizes() == 0).sum() == 90
    with pytest.raises(ValueError):
        s2.BlockPartition(5, 6)
    assert s2.sketch_cols(0.5, 0.01, 1_000_000) == 1667


def _build_c_smoke(tmp_path):
    """Compile tests/c/abi_smoke.c against include/s2.h and libs2.so with gcc (plain C99)."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    if gcc is None or not os.path.exists(os.path.join(cuda, "include", "cuda_runtime.h")):
        pytest.skip("gcc or CUDA headers missing")
    libdir = os.path.join(ROOT, "paper_2110_02140_b200")
    exe = str(tmp_path / "abi_smoke")
    cmd = [gcc, "-std=c99", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(cuda, "include"), os.path.join(ROOT, "tests", "c", "abi_smoke.c"),
           "-L" + libdir, "-ls2", "-L" + os.path.join(cuda, "lib64"), "-lcudart",
           "-Wl,-rpath," + libdir, "-Wl,-rpath," + os.path.join(cuda, "lib64"), "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_links_and_runs_host_entry_points(tmp_path):
    """The header is valid C99 and a C program links libs2.so with no Python or torch in the
    picture; its host-side entry points (hash KATs, plan validation errors) run here."""
    import subprocess

    exe = _build_c_smoke(tmp_path)
    r = subprocess.run([exe, "--no-gpu"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "abi_smoke ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_c_program_tiny_table_kat_on_gpu(tmp_path):
    """Plain C through the C ABI: SURVEY Appendix B tiny-table KAT (table rows, bitmap word,
    decode == input, counters, NaN flag) via s2_compress / s2_decode on cuda:0."""
    import subprocess

    exe = _build_c_smoke(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "abi_smoke ok" in r.stdout, r.stdout + r.stderr
