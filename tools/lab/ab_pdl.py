"""A/B of two builds of libgpuarray.so (tuning lab, GPU only) on the bench
step's five calls (axpbyz, dot, sum, norm2 into one device vector, exclusive
int32 scan) back to back, and on isolated calls after an L2 flush (the
tools/sweep.py protocol).  Both libraries are loaded in one process and the
timings interleave A, B, A, B so box and clock drift cancel.
    python tools/lab/ab_pdl.py LIB_A LIB_B [log2n ...]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1304_5553_b200 import _abi as A  # noqa: E402


def load(path):
    A.LIB_PATH = os.path.abspath(path)
    return A._load()


def main():
    libs = [load(sys.argv[1]), load(sys.argv[2])]
    lgs = [int(a) for a in sys.argv[3:]] or [14, 16, 18, 20, 22, 24, 26, 28]
    dev = torch.device("cuda:0")
    big = 1 << max(lgs)
    x, y = torch.rand(big, device=dev), torch.rand(big, device=dev)
    z = torch.empty_like(x)
    k = torch.randint(0, 10, (big,), dtype=torch.int32, device=dev)
    s_out = torch.empty_like(k)
    red = torch.zeros(3, dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.float32, device=dev)
    rws = [torch.zeros(lib.gpuarray_reduce_workspace_bytes(A.GA_F64, big), dtype=torch.uint8, device=dev)
           for lib in libs]
    sws = [torch.zeros(lib.gpuarray_scan_workspace_bytes(A.GA_I64, big), dtype=torch.uint8, device=dev)
           for lib in libs]
    st = torch.cuda.current_stream().cuda_stream
    a5, b6 = A.make_scalar(A.GA_F32, 5.0), A.make_scalar(A.GA_F32, 6.0)
    f = A.GA_F32

    def step(i, n, ops):
        lib, rw, sw = libs[i], rws[i], sws[i]
        if "axpbyz" in ops:
            assert lib.gpuarray_axpbyz(f, n, a5, x.data_ptr(), b6, y.data_ptr(), z.data_ptr(), st) == 0
        if "dot" in ops:
            assert lib.gpuarray_reduce(0, 1, f, f, n, x.data_ptr(), y.data_ptr(), red.data_ptr(), rw.data_ptr(),
                                       rw.numel(), st) == 0
        if "sum" in ops:
            assert lib.gpuarray_reduce(0, 0, f, f, n, x.data_ptr(), None, red.data_ptr() + 4, rw.data_ptr(),
                                       rw.numel(), st) == 0
        if "norm2" in ops:
            assert lib.gpuarray_reduce(0, 2, f, f, n, x.data_ptr(), None, red.data_ptr() + 8, rw.data_ptr(),
                                       rw.numel(), st) == 0
        if "scan" in ops:
            assert lib.gpuarray_scan(0, 1, A.GA_I32, A.GA_I32, n, k.data_ptr(), s_out.data_ptr(), None, 0,
                                     sw.data_ptr(), sw.numel(), st) == 0

    full = ("axpbyz", "dot", "sum", "norm2", "scan")
    for lg in lgs:
        n = 1 << lg
        for label, ops, iso in (("step x5", full, False), ("sum", ("sum",), False), ("sum iso", ("sum",), True),
                                ("norm2 iso", ("norm2",), True)):
            calls = 1 if iso else max(1, min(100, (1 << 26) // n))
            for i in (0, 1, 0, 1):
                step(i, n, ops)
            ts = [[], []]
            for _ in range(15):
                for i in (0, 1):
                    if iso:
                        flush.fill_(1.0)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(calls):
                        step(i, n, ops)
                    e1.record()
                    torch.cuda.synchronize()
                    ts[i].append(e0.elapsed_time(e1) * 1e3 / calls)
            a, b = statistics.median(ts[0]), statistics.median(ts[1])
            print(f"2^{lg} {label:10s} x{calls:<3d} A {a:9.2f} us  B {b:9.2f} us  A-B {a - b:+7.2f}", flush=True)


if __name__ == "__main__":
    main()
