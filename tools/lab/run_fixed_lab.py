"""Fixed per-call cost of the fp32 sum (tuning lab, GPU only): fixed_lab.cu
variants and the product sum at n = 2^22 .. 2^30, each call isolated (L2
flushed and cleaned as in tools/sweep.py) and back to back; the fixed cost F
and the streaming rate R come from a least-squares fit t = F + 4n / R over
2^26 .. 2^30.   python tools/lab/run_fixed_lab.py build | run"""
import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libfixed_lab.so")


def build():
    csrc = os.path.join(ROOT, "paper_1304_5553_b200", "csrc")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-I", csrc,
                           "-I", os.path.join(ROOT, "include"), "-o", LIB, os.path.join(HERE, "fixed_lab.cu")])


def main():
    import torch
    from paper_1304_5553_b200 import gpuarray as G
    L = ctypes.CDLL(LIB)
    L.fixed_lab.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    x = torch.rand(1 << 30, device=dev)
    part = torch.empty(1 << 20, device=dev)
    out = torch.empty((), device=dev)
    flush = torch.empty(512 << 20 >> 2, device=dev)
    clean = torch.ones(512 << 20 >> 2, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    names = {0: "empty kernel, same grid", 1: "loads only, no finish", 2: "loads only, persistent grid",
             9: "product sum (finish)"}
    lgs = list(range(22, 31))
    res = {}
    for v in names:
        for mode in ("isolated", "back-to-back"):
            ts = []
            for lg in lgs:
                n = 1 << lg
                def call():
                    if v == 9:
                        G.sum(x[:n], out=out)
                    else:
                        assert L.fixed_lab(v, n, x.data_ptr(), part.data_ptr(), s) == 0
                for _ in range(3):
                    call()
                reps, best = (1, []) if mode == "isolated" else (max(1, min(50, (1 << 28) // n)), [])
                for _ in range(11):
                    if mode == "isolated":
                        flush.fill_(1.0)
                        G.sum(clean, out=out)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(reps):
                        call()
                    e1.record()
                    torch.cuda.synchronize()
                    best.append(e0.elapsed_time(e1) * 1e3 / reps)
                ts.append(float(np.median(best)))
            res[(v, mode)] = ts
            fit = [i for i, lg in enumerate(lgs) if lg >= 26]
            A = np.array([[1.0, 4.0 * (1 << lgs[i])] for i in fit])
            F, inv = np.linalg.lstsq(A, np.array([ts[i] for i in fit]), rcond=None)[0]
            rate = 1e-3 / inv if inv > 0 else float("nan")
            print(f"{names[v]:32s} {mode:12s} " + " ".join(f"2^{lg}:{t:8.2f}" for lg, t in zip(lgs, ts))
                  + f"   fit F = {F:6.2f} us, R = {rate:6.0f} GB/s", flush=True)


if __name__ == "__main__":
    build() if sys.argv[1:] == ["build"] else main()
