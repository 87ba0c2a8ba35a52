"""Streaming ceilings of the scan's possible structures (tuning lab, GPU
only): struct_lab.cu variants at 1 GiB and 4 GiB (int32 2^28 / 2^30), back-
to-back calls, CUDA events, next to the product scan (gpuarray.scan).
    python tools/lab/run_struct_lab.py build | run [variants]"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libstruct_lab.so")


def build():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-o", LIB, os.path.join(HERE, "struct_lab.cu")])


def main():
    import torch
    from paper_1304_5553_b200 import gpuarray as G
    L = ctypes.CDLL(LIB)
    L.struct_lab.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_void_p]
    variants = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
        [60, 0, 1, 2, 3, 4, 5, 10, 11, 12, 13, 40, 41, 42, 43, 50, 51, 52, 53, 99]
    dev = torch.device("cuda:0")
    a = torch.randint(0, 10, (1 << 30,), dtype=torch.int32, device=dev)
    b = torch.empty(1 << 30, dtype=torch.int32, device=dev)
    sink = torch.zeros(64, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for lg in (28, 30):
        n = 1 << lg
        nbytes = 4 * n
        for v in variants:
            def call():
                if v == 99:
                    G.scan(a[:n], exclusive=True, out=b[:n])
                else:
                    rc = L.struct_lab(v, nbytes, a.data_ptr(), b.data_ptr(), sink.data_ptr(), s)
                    assert rc == 0, (v, rc)
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            res = []
            for _ in range(3):
                reps = 10
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    call()
                e1.record()
                torch.cuda.synchronize()
                res.append(e0.elapsed_time(e1) / reps * 1e3)
            us = min(res)
            print(f"2^{lg} variant {v:3d}  {us:8.1f} us ({max(res):8.1f})  {2 * nbytes / us / 1e3:7.1f} GB/s",
                  flush=True)


if __name__ == "__main__":
    build() if sys.argv[1:] == ["build"] else main()
