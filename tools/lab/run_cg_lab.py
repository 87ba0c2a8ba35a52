"""Fused CG kernel shapes (tuning lab, GPU only): time every variant of
cg_lab.cu at n = 2^20 .. 2^26 fp32 (back-to-back calls, working sets > L2
for n >= 2^24), GB/s of each kernel's algorithmic bytes (4 / 6 element-sizes).
    python tools/lab/run_cg_lab.py build | run"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libcg_lab.so")


def build():
    csrc = os.path.join(ROOT, "paper_1304_5553_b200", "csrc")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-I", csrc,
                           "-I", os.path.join(ROOT, "include"), "-o", LIB, os.path.join(HERE, "cg_lab.cu")])


def main():
    import torch
    L = ctypes.CDLL(LIB)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    L.lab_dir.argtypes = [ctypes.c_int, i64] + [vp] * 9
    L.lab_upd.argtypes = [ctypes.c_int, i64] + [vp] * 9
    dev = torch.device("cuda:0")
    s = torch.cuda.current_stream().cuda_stream
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    num = torch.tensor([0.5], device=dev)
    den = torch.tensor([2.0], device=dev)
    out = torch.zeros(1, device=dev)
    for lg in (20, 22, 24, 26):
        n = 1 << lg
        r, p, pout, ap, x = (torch.rand(n, device=dev) for _ in range(5))
        line = []
        for kind, fn, elts in (("dir", lambda v: L.lab_dir(v, n, r.data_ptr(), p.data_ptr(), pout.data_ptr(),
                                                               ap.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                                               num.data_ptr(), den.data_ptr(), s), 4),
                               ("upd", lambda v: L.lab_upd(v, n, x.data_ptr(), r.data_ptr(), pout.data_ptr(),
                                                           ap.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                                           num.data_ptr(), den.data_ptr(), s), 6)):
            for v in range(8):
                for _ in range(3):
                    rc = fn(v)
                torch.cuda.synchronize()
                if rc:
                    line.append(f"{kind}{v}:rc{rc}")
                    continue
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 20
                e0.record()
                for _ in range(reps):
                    fn(v)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / reps * 1e3
                line.append(f"{kind}{v}:{us:.1f}us/{elts * 4 * n / (us * 1e-6) / 1e9:.0f}")
        print(f"2^{lg}: " + "  ".join(line), flush=True)


if __name__ == "__main__":
    build() if len(sys.argv) > 1 and sys.argv[1] == "build" else main()
