"""Single-touch scan shapes against the product scan (tuning lab, GPU only):
smem_lab.cu variants at n = 2^lo..2^hi, back-to-back calls (inputs >= 4x L2
from 2^28; smaller n L2-warm), exact parity against the product scan.
    python tools/lab/run_smem_lab.py build | run lo hi [variants] [pf_dists]"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libsmem_lab.so")


def build():
    csrc = os.path.join(ROOT, "paper_1304_5553_b200", "csrc")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "--expt-relaxed-constexpr", "-Xptxas", "-v", "-Xcompiler", "-fPIC", "-shared", "-I", csrc, "-I", HERE,
                           "-I", os.path.join(ROOT, "include"), "-o", LIB, os.path.join(HERE, "smem_lab.cu")])


def main():
    import torch
    from paper_1304_5553_b200 import gpuarray as G
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    variants = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0, 1, 2, 3, 4, 5, 6, 7, 10, 11, 12, 13]
    pfds = [int(v) for v in sys.argv[5].split(",")] if len(sys.argv) > 5 else [148]
    L = ctypes.CDLL(LIB)
    L.smem_lab.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    N = 1 << hi
    k32 = torch.randint(0, 10, (N,), dtype=torch.int32, device=dev)
    k64 = torch.randint(0, 10, (N,), dtype=torch.int64, device=dev) if any(v >= 20 for v in variants) else None
    o32 = torch.empty_like(k32)
    o64 = torch.empty_like(k64) if k64 is not None else None
    ws = torch.zeros(256 + 16 * (N // 1024) + (1 << 20), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for lg in range(lo, hi + 1):
        n = 1 << lg
        reps = max(3, min(50, (1 << 28) // n))
        for ex in (1,):
            line = []
            cands = [(-1, 0)] + [(v, d) for v in variants for d in (pfds if v in (10, 11, 12, 13, 23) else [0])]
            for v, d in cands:
                is64 = 20 <= v < 30
                src, out = (k64[:n], o64[:n]) if is64 else (k32[:n], o32[:n])
                def call():
                    if v < 0:
                        G.scan(src, exclusive=bool(ex), out=out)
                    else:
                        rc = L.smem_lab(v, ex, n, src.data_ptr(), out.data_ptr(), ws.data_ptr(), d, s)
                        assert rc == 0, (v, rc)
                call()
                torch.cuda.synchronize()
                ok = v < 0 or torch.equal(out, G.scan(src, exclusive=bool(ex)))
                for _ in range(2):
                    call()
                best = 1e30
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(reps):
                        call()
                    e1.record()
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1) / reps * 1e3)
                gbs = 2 * n * (8 if is64 else 4) / (best * 1e-6) / 1e9
                tag = "prod" if v < 0 else f"{v}" + (f"@{d}" if d else "")
                line.append(f"{tag}:{best:.1f}us/{gbs:.0f}{'' if ok else '!FAIL'}")
            print(f"2^{lg} ex={ex}: " + "  ".join(line), flush=True)


if __name__ == "__main__":
    build() if sys.argv[1:] == ["build"] else main()
