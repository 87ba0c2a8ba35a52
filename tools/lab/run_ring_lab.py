"""Register-held single-touch scan (ring_lab.cu) against the product scan
(tuning lab, GPU only): int32 SUM, back-to-back calls, exact parity against
the product scan, CUDA events.
    python tools/lab/run_ring_lab.py build | run lo hi [variants]"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libring_lab.so")


def build():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xptxas", "-v", "-Xcompiler", "-fPIC", "-shared", "-o", LIB,
                           os.path.join(HERE, "ring_lab.cu")])


def main():
    import torch
    from paper_1304_5553_b200 import gpuarray as G
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    variants = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else list(range(10))
    L = ctypes.CDLL(LIB)
    L.ring_lab.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    N = 1 << hi
    k32 = torch.randint(0, 10, (N,), dtype=torch.int32, device=dev)
    o32 = torch.empty_like(k32)
    status = torch.zeros(N // 1024 + 1024, dtype=torch.int64, device=dev)
    tickets = torch.zeros(1 << 16, dtype=torch.int64, device=dev)
    epoch = [0]
    s = torch.cuda.current_stream().cuda_stream
    for lg in range(lo, hi + 1):
        n = 1 << lg
        reps = max(3, min(50, (1 << 28) // n))
        for ex in (1, 0):
            ref = G.scan(k32[:n], exclusive=bool(ex))
            line = []
            for v in [-1] + variants:
                src, out = k32[:n], o32[:n]

                def call():
                    if v < 0:
                        G.scan(src, exclusive=bool(ex), out=out)
                    else:
                        epoch[0] += 1
                        assert epoch[0] < (1 << 16)
                        rc = L.ring_lab(v, ex, n, src.data_ptr(), out.data_ptr(), status.data_ptr(),
                                        tickets[epoch[0]:].data_ptr(), epoch[0], s)
                        assert rc == 0, (v, rc)
                if v >= 0 and n % L.ring_lab_tile_elems(v):
                    line.append(f"{v}:n/a")
                    continue
                out.zero_()
                call()
                torch.cuda.synchronize()
                ok = torch.equal(out, ref)
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
                gbs = 2 * n * 4 / (best * 1e-6) / 1e9
                tag = "prod" if v < 0 else f"{v}"
                line.append(f"{tag}:{best:.1f}us/{gbs:.0f}{'' if ok else '!FAIL'}")
            print(f"2^{lg} ex={ex}: " + "  ".join(line), flush=True)


def trace():
    """python run_ring_lab.py trace v lg: one traced exclusive call after warm-up; per-tile phase times."""
    import numpy as np
    import torch
    v, lg = int(sys.argv[2]), int(sys.argv[3])
    L = ctypes.CDLL(LIB)
    L.ring_lab_trace.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    n = 1 << lg
    k32 = torch.randint(0, 10, (n,), dtype=torch.int32, device=dev)
    o32 = torch.empty_like(k32)
    status = torch.zeros(n // 1024 + 1024, dtype=torch.int64, device=dev)
    tickets = torch.zeros(64, dtype=torch.int64, device=dev)
    te = L.ring_lab_tile_elems(v)
    nt = n // te
    tr = torch.zeros(nt * 8, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for e in range(1, 6):
        assert L.ring_lab_trace(v, n, k32.data_ptr(), o32.data_ptr(), status.data_ptr(), tickets[e:].data_ptr(), e,
                                tr.data_ptr() if e == 5 else None, s) == 0
    torch.cuda.synchronize()
    a = tr.view(-1, 8).cpu().numpy().astype(np.int64)
    a = a - a[:, 0].min()
    names = ["issue", "landed", "agg pub", "lb start", "prefix", "data lds", "data pref", "data stored"]
    print(f"v={v} 2^{lg}: {nt} tiles, span {a[:, 7].max() / 1e3:.1f} us")
    for i in range(1, 8):
        d = (a[:, i] - a[:, i - 1]) / 1e3
        print(f"  {names[i - 1]:>10} -> {names[i]:<11} mean {d.mean():6.2f} p50 {np.median(d):6.2f} p90 {np.percentile(d, 90):6.2f} us")
    d = (a[:, 7] - a[:, 0]) / 1e3
    print(f"  life mean {d.mean():.2f} us; landed->prefix {((a[:, 4] - a[:, 1]) / 1e3).mean():.2f}")
    # predecessor lag: latest aggregate among the 256 previous tiles vs this tile's
    lag = []
    for t in range(300, nt, 7):
        lag.append((a[t - 256:t, 2].max() - a[t, 2]) / 1e3)
    print(f"  latest predecessor agg after own: mean {np.mean(lag):.2f} p90 {np.percentile(lag, 90):.2f} us")
    mid = a[:, 7].max() // 2
    print("  tiles alive at mid-run by phase:", [int(((a[:, i] <= mid) & (a[:, i + 1] > mid)).sum()) for i in range(7)])


if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:
        build()
    elif sys.argv[1] == "trace":
        trace()
    else:
        main()
