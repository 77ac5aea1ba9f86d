"""Build libs2.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with gpurun).

    python paper_2110_02140_b200/build.py [--force]
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libs2.so")
SOURCES = ["s2_compress.cu", "s2_decode.cu", "s2_kernels.cu", "s2_p2p.cu", "s2_topk.cu", "s2_capi.cu"]
HEADERS = ["s2_common.cuh", "s2_kernels.h", "s2_decode.cuh", "s2_device.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    """NCCL headers + lib from the torch-bundled nvidia-nccl wheel (the same libnccl.so.2 torch loads)."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl.h not found in the nvidia-nccl wheel")


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "s2.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = True) -> str:
    """Compile each .cu to an object in parallel (the kernels are template-heavy), then link."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    inc, lib = nccl_dirs()
    objdir = os.path.join(PKG, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    extra = os.environ.get("S2_NVCC_FLAGS", "").split()
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *extra,
              "-Xptxas", "-v" if verbose and os.environ.get("S2_PTXAS_V") else "-O3",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = common + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.stdout or r.stderr:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise subprocess.CalledProcessError(r.returncode, cmd)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    link = [nvcc(), *ARCH, "-shared", *objs, "-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}",
            "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
