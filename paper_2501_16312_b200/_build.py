"""Build liblinprim.so in-tree with nvcc for sm_100a (B200)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "liblinprim.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-O3"]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(os.path.join(PKG, "csrc", "*.h")) + \
        [os.path.join(ROOT, "include", "linprim.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    """variant "checked": liblinprim_checked.so with the device-side bounds checks (-DLP_CHECKED),
    loaded only when LP_LIB points at it (tests/test_gpu_checked.py)."""
    lib = LIB if not variant else os.path.join(PKG, f"liblinprim_{variant}.so")
    if force or not os.path.exists(lib) or any(os.path.getmtime(d) > os.path.getmtime(lib) for d in _deps()):
        nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
        extra = os.environ.get("LP_EXTRA_NVCC_FLAGS", "").split()   # measurement variants only
        if variant == "checked":
            extra = extra + ["-DLP_CHECKED"]
        cmd = [nvcc] + NVCC_FLAGS + extra + ["-o", lib + ".tmp"] + sources()
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        os.replace(lib + ".tmp", lib)
    return lib
