"""Compile the product library libgpuarray.so for sm_100a (nvcc, in-tree).

    python paper_1304_5553_b200/build.py [--force]

Run as a file (or loaded by path, see __graft_entry__.py / tests/conftest.py):
importing the package itself loads libgpuarray.so, which may be the stale
library this script is about to replace.

Only the product sources (csrc/*.cu + include/gpuarray.h) are compiled here.
The CPU oracle and the synthetic generator have their own build steps
(__graft_entry__.build())."""
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libgpuarray.so")
SOURCES = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
DEPS = SOURCES + glob.glob(os.path.join(PKG, "csrc", "*.h")) + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + \
    [os.path.join(ROOT, "include", "gpuarray.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "static",
]


def nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp", *SOURCES]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
