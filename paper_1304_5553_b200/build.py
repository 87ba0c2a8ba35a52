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


def nccl_include():
    """nccl.h for the sharded entry points (types only: NCCL is bound at run
    time with dlopen).  The NCCL wheel torch links against, else the system's."""
    import sysconfig
    cand = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl", "include")
    return cand if os.path.exists(os.path.join(cand, "nccl.h")) else "/usr/include"


def nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force=False, verbose=False):
    """Compile every csrc/*.cu to an object in parallel, then link."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared",)]
    jobs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        jobs.append((obj, [nvcc(), *compile_flags, "-I", os.path.join(ROOT, "include"), "-I", nccl_include(),
                           "-c", "-o", obj, src]))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
        for obj, cmd in jobs:
            if verbose:
                print(" ".join(cmd), flush=True)
        list(ex.map(lambda j: subprocess.check_call(j[1]), jobs))
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
            "-o", LIB + ".tmp", *[o for o, _ in jobs], "-ldl"]
    subprocess.check_call(link)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
