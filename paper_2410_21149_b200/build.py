"""Build libcvx.so (the C-ABI library, include/cvx.h) for sm_100a with nvcc, in-tree."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcvx.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-shared", "--cudart", "static",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "cvx.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp", *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


BOUNDS_LIB = os.path.join(HERE, "libcvx_bounds.so")


def build_bounds(force: bool = False) -> str:
    """The same library with the device-side bounds checks of CVX_BOUNDS=1 (cvx_internal.cuh)."""
    if not force and os.path.exists(BOUNDS_LIB) and all(os.path.getmtime(d) <= os.path.getmtime(BOUNDS_LIB) for d in deps()):
        return BOUNDS_LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-DCVX_BOUNDS=1", "-I", os.path.join(ROOT, "include"), "-o", BOUNDS_LIB + ".tmp", *sources()]
    subprocess.check_call(cmd)
    os.replace(BOUNDS_LIB + ".tmp", BOUNDS_LIB)
    return BOUNDS_LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
