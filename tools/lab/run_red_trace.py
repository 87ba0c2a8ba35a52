"""Timeline of a one-shot streaming reduction (tuning lab, GPU only): per-CTA
globaltimer stamps from red_trace_lab.cu -> kernel span vs CUDA-event time,
ramp-up, tail, and delivered bandwidth per microsecond bucket.
    python tools/lab/run_red_trace.py build | [log2n ...]"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libred_trace_lab.so")


def build():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-o", LIB, os.path.join(HERE, "red_trace_lab.cu")])


def main(lgs):
    import numpy as np
    import torch
    L = ctypes.CDLL(LIB)
    L.red_trace.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 6
    dev = torch.device("cuda:0")
    x = torch.rand(1 << max(lgs), device=dev)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
    out = torch.zeros(1, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for lg in lgs:
        n = 1 << lg
        grid = n // 4 // (256 * 16)
        tr = torch.zeros(grid * 4, dtype=torch.int64, device=dev)
        args = lambda: (n, x.data_ptr(), ws.data_ptr() + 128, ws.data_ptr(), out.data_ptr(), tr.data_ptr(), s)  # noqa
        for _ in range(5):
            L.red_trace(*args())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            L.red_trace(*args())
        e1.record()
        torch.cuda.synchronize()
        ev_us = e0.elapsed_time(e1) / reps * 1e3
        t = tr.view(grid, 4).cpu().numpy()
        t0 = t[:, 0].min()
        st, ld, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
        span = en.max()
        life = en - st
        sms = len(set(t[:, 3].tolist()))
        nbytes = 4 * n
        print(f"2^{lg}: grid {grid}  event {ev_us:.1f} us ({nbytes / ev_us / 1e3:.0f} GB/s)  span {span:.1f} us "
              f"({nbytes / span / 1e3:.0f} GB/s)  SMs {sms}")
        print(f"   CTA life p10/p50/p90/max {np.percentile(life, 10):.2f}/{np.median(life):.2f}/"
              f"{np.percentile(life, 90):.2f}/{life.max():.2f} us; finish (end - loads back) p50 "
              f"{np.median(en - ld):.2f} max {(en - ld).max():.2f}")
        first_wave = np.sort(st)[min(sms * 4, grid) - 1]
        print(f"   first {min(sms * 4, grid)} CTAs started by {first_wave:.2f} us; last CTA start {st.max():.2f}; "
              f"last load back {ld.max():.2f}; last end {en.max():.2f}")
        per = nbytes / grid
        hist, edges = np.histogram(ld, bins=np.arange(0, span + 2, 2.0))
        bw = hist * per / 2e-6 / 1e9
        head = " ".join(f"{b:.0f}" for b in bw[:6])
        tail = " ".join(f"{b:.0f}" for b in bw[-6:])
        mid = np.median(bw[3:-3]) if len(bw) > 8 else float("nan")
        print(f"   GB/s per 2us bucket: head [{head}]  mid {mid:.0f}  tail [{tail}]")


if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:
        build()
    else:
        main([int(a) for a in sys.argv[1:]] or [24, 26, 28, 30])
