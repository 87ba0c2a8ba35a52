"""1:1 copy / write-only HBM ceilings (tuning lab, GPU only): copy_lab.cu
variants at 2^28 and 2^30 int32-equivalent sizes, back-to-back calls, CUDA
events; torch copy_ (variant 99) beside them.
    python tools/lab/run_copy_lab.py build | run"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libcopy_lab.so")


def build():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-o", LIB, os.path.join(HERE, "copy_lab.cu")])


def main():
    import torch
    L = ctypes.CDLL(LIB)
    L.copy_lab.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    a = torch.ones(2 << 30, dtype=torch.int32, device=dev)  # mix21 reads a[:n] and a[n:2n]
    b = torch.empty(1 << 30, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for lg in (28, 30):
        nbytes = 4 << lg
        for v in (0, 1, 2, 3, 4, 5, 10, 11, 20, 21, 22, 23, 99):
            def call():
                if v == 99:
                    b[: nbytes // 4].copy_(a[: nbytes // 4])
                else:
                    assert L.copy_lab(v, nbytes, a.data_ptr(), b.data_ptr(), s) == 0
            for _ in range(3):
                call()
            reps = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                call()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / reps * 1e3
            traffic = nbytes * (1 if v in (10, 11) else 3 if v >= 20 and v < 99 else 2)
            print(f"2^{lg} int32  variant {v:2d}  {us:8.1f} us  {traffic / us / 1e3:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    build() if sys.argv[1:] == ["build"] else main()
