"""Scan super-tile shape vs n (tuning lab, GPU only): every variant of
tile_lab.cu at n = 2^lo .. 2^hi, one call per timing with the L2 flushed
before it (the tools/sweep.py protocol), parity against the product scan.
    python tools/lab/run_tile_lab.py build | [lo hi]"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.environ.get("TILE_LAB_LIB", os.path.join(HERE, "libtile_lab.so"))


def build():
    csrc = os.path.join(ROOT, "paper_1304_5553_b200", "csrc")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-I", csrc,
                           "-I", os.path.join(ROOT, "include"), "-o", LIB, os.path.join(HERE, "tile_lab.cu")])


def main():
    import torch
    import synth
    from paper_1304_5553_b200 import gpuarray as G
    lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (18, 28)
    variants = [int(v) for v in os.environ.get("TILE_LAB_VARIANTS", "0,1,2,3,4,5,6,7,8,9,10,11,12,20,21,22,23,24").split(",")]
    L = ctypes.CDLL(LIB)
    if os.environ.get("PERSIST_L2_MB"):
        L.lab_set_persisting_l2.argtypes = [ctypes.c_size_t]
        print("persisting L2 carve-out MiB:", L.lab_set_persisting_l2(int(os.environ["PERSIST_L2_MB"]) << 20),
              flush=True)
    L.lab_scan.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p]
    L.lab_scan_tile.restype = ctypes.c_int64
    dev = torch.device("cuda:0")
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    clean = torch.ones(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    sink = torch.empty((), dtype=torch.float32, device=dev)
    N = 1 << hi
    k32 = synth.device_fill(synth.I32_RANGE, 3, N, lo=0, hi=9, device=dev)
    need64 = any(L.lab_scan_elem_bytes(v) == 8 for v in variants)
    k64 = synth.device_fill(synth.I64_RANGE, 3, N, lo=0, hi=9, device=dev) if need64 else None
    o32 = torch.empty_like(k32)
    o64 = torch.empty_like(k64) if need64 else None
    ws = torch.zeros(256 + 32 * (N // 4096) + (1 << 20), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for lg in range(lo, hi + 1):
        n = 1 << lg
        best = None
        line = []
        for v in variants:
            is64 = L.lab_scan_elem_bytes(v) == 8
            src, out = (k64[:n], o64[:n]) if is64 else (k32[:n], o32[:n])
            ws.zero_()
            for _ in range(3):
                rc = L.lab_scan(v, n, src.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
            if rc:
                line.append(f"{v}:rc{rc}")
                continue
            torch.cuda.synchronize()
            ok = torch.equal(out, G.scan(src, exclusive=True))
            ts = []
            for _ in range(15):
                flush.fill_(1.0)
                G.sum(clean, out=sink)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                L.lab_scan(v, n, src.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            us = ts[len(ts) // 2] * 1e3
            gbs = 2 * n * (8 if is64 else 4) / (us * 1e-6) / 1e9
            line.append(f"{v}:{us:.1f}us/{gbs:.0f}{'' if ok else '!FAIL'}")
        print(f"2^{lg}: " + "  ".join(line), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "build":
        build()
    else:
        main()
