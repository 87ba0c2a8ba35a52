"""A/B of two builds of libgpuarray.so on gpuarray_scan (tuning lab, GPU
only): both libraries loaded in one process, calls interleaved, back-to-back
calls between one event pair per (lib, rep), median over reps.
    python tools/lab/ab_scan.py LIB_A LIB_B [log2n ...]"""
import ctypes
import statistics
import sys

import torch

GA_F32, GA_F64, GA_I32, GA_I64 = 0, 1, 2, 3
SUM = 0
INCL, EXCL = 0, 1


def load(path):
    lib = ctypes.CDLL(path)
    lib.gpuarray_scan.restype = ctypes.c_int
    lib.gpuarray_scan.argtypes = [ctypes.c_int] * 4 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                                       ctypes.c_size_t, ctypes.c_void_p]
    lib.gpuarray_scan_workspace_bytes.restype = ctypes.c_size_t
    lib.gpuarray_scan_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int64]
    return lib


def main():
    libs = [load(sys.argv[1]), load(sys.argv[2])]
    lgs = [int(a) for a in sys.argv[3:]] or [20, 24, 28, 30]
    dev = torch.device("cuda:0")
    big = 1 << max(lgs)
    k32 = torch.randint(0, 10, (big,), dtype=torch.int32, device=dev)
    k64 = torch.randint(0, 10, (big,), dtype=torch.int64, device=dev)
    f32 = torch.rand(big, device=dev)
    o64 = torch.empty(big, dtype=torch.int64, device=dev)
    o32 = torch.empty_like(k32)
    wss = [torch.zeros(lib.gpuarray_scan_workspace_bytes(GA_I64, big) + 4096, dtype=torch.uint8, device=dev)
           for lib in libs]
    s = torch.cuda.current_stream().cuda_stream
    cases = [("i32 incl", GA_I32, GA_I32, INCL, k32, o32), ("i32 excl", GA_I32, GA_I32, EXCL, k32, o32),
             ("i64 incl", GA_I64, GA_I64, INCL, k64, o64), ("i64 excl", GA_I64, GA_I64, EXCL, k64, o64),
             ("i32>i64 in", GA_I32, GA_I64, INCL, k32, o64), ("f32>f64 in", GA_F32, GA_F64, INCL, f32, o64)]
    for lg in lgs:
        for name, idt, odt, kind, x, o in cases:
            n = 1 << lg
            calls = max(1, min(50, (1 << 26) // n))
            outs = [None, None]

            def run(i):
                lib, ws = libs[i], wss[i]
                for _ in range(calls):
                    rc = lib.gpuarray_scan(SUM, kind, idt, odt, n, x.data_ptr(), o.data_ptr(), None, 0,
                                           ws.data_ptr(), ws.numel(), s)
                    assert rc == 0, rc
            for i in (0, 1):
                run(i)
                torch.cuda.synchronize()
                outs[i] = o[:n].clone() if lg <= 28 else o[:1 << 20].clone()
            same = torch.equal(outs[0], outs[1])
            ts = [[], []]
            for _ in range(11):
                for i in (0, 1):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    run(i)
                    e1.record()
                    torch.cuda.synchronize()
                    ts[i].append(e0.elapsed_time(e1) * 1e3 / calls)
            a, b = statistics.median(ts[0]), statistics.median(ts[1])
            print(f"2^{lg} {name:10s} x{calls:<3d} A {a:9.2f} us  B {b:9.2f} us  A-B {a - b:+7.2f}"
                  f"  {'same' if same else 'DIFF'}", flush=True)


if __name__ == "__main__":
    main()
