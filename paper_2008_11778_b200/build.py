"""Build libseisgpu.so in-tree with nvcc for sm_100a.

    python -m paper_2008_11778_b200.build

The shared library is the product: hand-written CUDA kernels plus the C ABI
declared in include/seisgpu.h.  cudart is linked statically (nvcc default), so
the library does not depend on the CUDA runtime version torch ships.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libseisgpu.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def needs_rebuild():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + [
        os.path.join(ROOT, "include", "seisgpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, out=None, defines=()):
    """Compile csrc/*.cu into `out` (default: the in-tree libseisgpu.so)."""
    lib = out or LIB
    if out is None and not force and not needs_rebuild():
        return LIB
    nvcc = nvcc_path()
    cmd = [nvcc, "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O3",
           "-shared", "-I", os.path.join(ROOT, "include"), *[f"-D{d}" for d in defines],
           "-o", lib + ".tmp", *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
