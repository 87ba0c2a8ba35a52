"""Reduction CTA shape at large n (tuning lab, GPU only): red_shape_lab.cu
variants, back-to-back calls between one event pair, median of 15, fp32,
interleaved so drift cancels.
    RED_LAB_LIB=libred_shape.so RED_LAB_SRC=red_shape_lab.cu python tools/lab/run_red_lab.py build
    VARIANTS=3,5 python tools/lab/run_red_large.py [log2n ...]"""
import ctypes
import os
import statistics
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    import torch
    L = ctypes.CDLL(os.path.join(HERE, "libred_shape.so"))
    L.red_lab.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 5
    dev = torch.device("cuda:0")
    lgs = [int(a) for a in sys.argv[1:]] or [26, 28, 30]
    x = torch.rand(1 << max(lgs), device=dev)
    y = torch.rand(1 << max(lgs), device=dev)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
    out = torch.empty(1, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    variants = [int(v) for v in os.environ.get("VARIANTS", "3,4,5,13,14,15,18").split(",")]
    for lg in lgs:
        n = 1 << lg
        calls = max(1, (1 << 28) // n)
        ts = {v: [] for v in variants}
        for rep in range(16):
            for v in variants:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(calls):
                    L.red_lab(v, n, x.data_ptr(), y.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
                e1.record()
                torch.cuda.synchronize()
                if rep:
                    ts[v].append(e0.elapsed_time(e1) * 1e3 / calls)
        print(f"2^{lg}: " + "  ".join(f"{v}:{statistics.median(ts[v]):.1f}" for v in variants), flush=True)


if __name__ == "__main__":
    main()
