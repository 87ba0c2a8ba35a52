"""A/B of two builds of libgpuarray.so on gpuarray_reduce (tuning lab, GPU
only): both libraries loaded in one process, calls interleaved A, B, A, B...
so box-to-box and clock drift cancel; back-to-back calls between one event
pair per (lib, rep), median over reps.
    python tools/lab/ab_reduce.py LIB_A LIB_B [log2n ...]
Build B from another revision with, e.g.:
    git worktree add /tmp/rev HEAD~1 && (cd /tmp/rev && python -c "import __graft_entry__ as g; g.build()")"""
import ctypes
import statistics
import sys

import torch

GA_F32, GA_F64 = 0, 1
SUM = 0
MAP_ID, MAP_MUL, MAP_SQ = 0, 1, 2


def load(path):
    lib = ctypes.CDLL(path)
    lib.gpuarray_reduce.restype = ctypes.c_int
    lib.gpuarray_reduce.argtypes = [ctypes.c_int] * 4 + [ctypes.c_int64] + [ctypes.c_void_p] * 4 + [ctypes.c_size_t,
                                                                                                    ctypes.c_void_p]
    lib.gpuarray_reduce_workspace_bytes.restype = ctypes.c_size_t
    lib.gpuarray_reduce_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int64]
    return lib


def main():
    libs = [load(sys.argv[1]), load(sys.argv[2])]
    lgs = [int(a) for a in sys.argv[3:]] or [20, 22, 24, 26, 28, 30]
    dev = torch.device("cuda:0")
    big = 1 << max(lgs)
    x32, y32 = torch.rand(big, device=dev), torch.rand(big, device=dev)
    x64 = torch.rand(big // 2 if max(lgs) >= 30 else big, device=dev, dtype=torch.float64)
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    wss = [torch.zeros(lib.gpuarray_reduce_workspace_bytes(GA_F64, big), dtype=torch.uint8, device=dev) for lib in libs]
    s = torch.cuda.current_stream().cuda_stream
    cases = [("sum f32", GA_F32, MAP_ID, x32, None), ("dot f32", GA_F32, MAP_MUL, x32, y32),
             ("norm2 f64", GA_F64, MAP_SQ, x64, None)]
    for lg in lgs:
        for name, dt, mp, x, y in cases:
            n = min(1 << lg, x.numel())
            calls = max(1, min(50, (1 << 26) // n))

            def run(i):
                lib, ws = libs[i], wss[i]
                for _ in range(calls):
                    rc = lib.gpuarray_reduce(SUM, mp, dt, dt, n, x.data_ptr(), y.data_ptr() if y is not None else None,
                                             out.data_ptr(), ws.data_ptr(), ws.numel(), s)
                    assert rc == 0, rc
            for i in (0, 1, 0, 1):
                run(i)
            ts = [[], []]
            for _ in range(15):
                for i in (0, 1):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    run(i)
                    e1.record()
                    torch.cuda.synchronize()
                    ts[i].append(e0.elapsed_time(e1) * 1e3 / calls)
            a, b = statistics.median(ts[0]), statistics.median(ts[1])
            print(f"2^{lg} {name:9s} x{calls:<3d} A {a:9.2f} us  B {b:9.2f} us  A-B {a - b:+7.2f}", flush=True)


if __name__ == "__main__":
    main()
