"""Time scan tile-shape variants side by side (tuning lab, GPU only).
    python tools/lab/run_scan_lab.py [log2n]"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, os.environ.get("SCAN_LAB_LIB", "libscan_lab.so"))
SRC = os.environ.get("SCAN_LAB_SRC", "scan_lab.cu")


def build():
    src = os.path.join(HERE, SRC)
    csrc = os.path.join(ROOT, "paper_1304_5553_b200", "csrc")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-I", csrc, "-I", HERE,
                           "-I", os.path.join(ROOT, "include"), "-o", LIB, src])


def main():
    import torch
    import synth
    from paper_1304_5553_b200 import gpuarray as G
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    only = [int(a) for a in sys.argv[2:]]
    variants = [int(v) for v in os.environ["SCAN_LAB_VARIANTS"].split(",")] if "SCAN_LAB_VARIANTS" in os.environ else None
    if not os.path.exists(LIB):
        build()
    L = ctypes.CDLL(LIB)
    L.lab_scan.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p]
    L.lab_scan_tile.restype = ctypes.c_int64
    n = 1 << lg
    dev = torch.device("cuda:0")
    k32 = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=dev)
    k64 = synth.device_fill(synth.I64_RANGE, 3, n, lo=0, hi=9, device=dev)
    ref32 = G.scan(k32, exclusive=True)
    ref64 = G.scan(k64, exclusive=True)
    o32, o64 = torch.empty_like(k32), torch.empty_like(k64)
    ws = torch.zeros(256 + 32 * n // 64 + (1 << 20), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for v in variants or [142, 232, 161] + list(range(240, 250)):
        if only and v not in only:
            continue
        is64 = L.lab_scan_elem_bytes(v) == 8
        src, out, ref = (k64, o64, ref64) if is64 else (k32, o32, ref32)
        ws.zero_()
        for _ in range(3):
            rc = L.lab_scan(v, n, src.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
            if rc != 0:
                break
        if rc != 0:
            print(f"variant {v:2d} launch failed rc={rc}", flush=True)
            continue
        torch.cuda.synchronize()
        ok = torch.equal(out, ref)
        reps = 20
        e0.record()
        for _ in range(reps):
            L.lab_scan(v, n, src.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = 2 * n * (8 if is64 else 4) / (ms * 1e-3) / 1e9
        for m in (1, 1000, 100003, 4 * 2048 * 7 + 5, n - 12345):
            ws.zero_()
            sub, osub = src[:m], out[:m]
            L.lab_scan(v, m, sub.data_ptr(), osub.data_ptr(), ws.data_ptr(), s)
            L.lab_scan(v, m, sub.data_ptr(), osub.data_ptr(), ws.data_ptr(), s)  # reuse (epoch)
            ok = ok and torch.equal(osub, G.scan(sub, exclusive=True))
        print(f"variant {v:2d} tile {L.lab_scan_tile(v):6d} {'i64' if is64 else 'i32'}  {ms*1e3:8.1f} us  "
              f"{gbs:7.1f} GB/s  parity={'ok' if ok else 'FAIL'}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "build":
        build()
    else:
        main()
