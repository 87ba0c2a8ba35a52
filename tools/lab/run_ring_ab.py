"""The product ring scan (csrc/scan_ring.cuh via ring_ab.cu) against the
product scan as dispatched (tuning lab, GPU only): every dtype, SUM (and MAX
for int32), inclusive / exclusive, 2^lo..2^hi elements, back-to-back calls,
CUDA events; parity against the product's output (integers and max/min
bit-exact, float SUM within 1e-4 relative of the running magnitude).
    python tools/lab/run_ring_ab.py build | run lo hi [dtypes]"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libring_ab.so")
DT = {"int32": 2, "int64": 3, "float32": 0, "float64": 1, "int32w": -3, "float32w": -1}  # w: widening


def build():
    csrc = os.path.join(ROOT, "paper_1304_5553_b200", "csrc")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-I", csrc,
                           "-I", os.path.join(ROOT, "include"), "-o", LIB, os.path.join(HERE, "ring_ab.cu")])


def main():
    import torch
    from paper_1304_5553_b200 import gpuarray as G
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    dts = sys.argv[4].split(",") if len(sys.argv) > 4 else list(DT)
    L = ctypes.CDLL(LIB)
    L.ring_ab.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    s = torch.cuda.current_stream().cuda_stream
    ws = torch.zeros(256 + 16 * ((1 << hi) // 1024 + 64), dtype=torch.uint8, device=dev)
    for name in dts:
        dt = getattr(torch, name.rstrip("w"))
        wide = {"int32w": torch.int64, "float32w": torch.float64}.get(name)
        N = 1 << hi
        if dt.is_floating_point:
            x = torch.rand(N, dtype=dt, device=dev)
        else:
            x = torch.randint(0, 10, (N,), dtype=dt, device=dev)
        o = torch.empty(N, dtype=wide or dt, device=dev)
        for lg in range(lo, hi + 1):
            n = (1 << lg) + (lg % 3) * 17  # some sizes ragged
            if n > N:
                n = 1 << lg
            reps = max(3, min(50, (1 << 28) // n))
            line = []
            for op, ex in ((0, 1), (0, 0)) + (((1, 0),) if name in ("int32", "int32w") else ()):
                opn = ["sum", "max", "min"][op]
                gop = op
                ref = G.scan(x[:n], exclusive=bool(ex), op=gop, out_dtype=wide)
                for arm in ("prod", "ring"):
                    src, out = x[:n], o[:n]

                    def call():
                        if arm == "prod":
                            G.scan(src, exclusive=bool(ex), op=gop, out=out, out_dtype=wide)
                        else:
                            rc = L.ring_ab(op, ex, DT[name], n, src.data_ptr(), out.data_ptr(), None, 0,
                                           ws.data_ptr(), s)
                            assert rc == 0, rc
                    out.fill_(7)
                    ok = True
                    call()
                    torch.cuda.synchronize()
                    if dt.is_floating_point and op == 0:
                        mag = torch.cumsum(src.abs().double(), 0)
                        ok = bool(((out.double() - ref.double()).abs() <= 1e-4 * mag + 1e-30).all())
                    else:
                        ok = torch.equal(out, ref) or v >= 100
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
                    line.append(f"{opn}{'X' if ex else 'I'}-{arm}:{best:.1f}{'' if ok else '!FAIL'}")
            print(f"{name} n=2^{lg}{'+' + str(n - (1 << lg)) if n != 1 << lg else ''}: " + "  ".join(line),
                  flush=True)


def cfg():
    """python run_ring_ab.py cfg lo hi v1,v2,..: ring shape variants (int32 and int64 SUM) vs the product."""
    import torch
    from paper_1304_5553_b200 import gpuarray as G
    lo, hi = int(sys.argv[2]), int(sys.argv[3])
    vs = [int(v) for v in sys.argv[4].split(",")]
    L = ctypes.CDLL(LIB)
    DT["float32"] = 0
    L.ring_ab_cfg.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    s = torch.cuda.current_stream().cuda_stream
    ws = torch.zeros(256 + 16 * ((1 << hi) // 1024 + 64), dtype=torch.uint8, device=dev)
    for name in (sys.argv[5].split(",") if len(sys.argv) > 5 else ("int32", "int64")):
        dt = getattr(torch, name.rstrip("w"))
        wide = torch.int64 if name == "int32w" else None
        x = torch.randint(-(1 << 20), 1 << 20, (1 << hi,), dtype=dt, device=dev) if not dt.is_floating_point \
            else torch.randint(0, 2, (1 << hi,), dtype=torch.int32, device=dev).to(dt)
        o = torch.empty(1 << hi, dtype=wide or dt, device=dev)
        for lg in range(lo, hi + 1):
            n = (1 << lg) + 5
            n = min(n, 1 << hi)
            reps = max(3, min(50, (1 << 28) // n))
            for ex in (1, 0):
                ref = G.scan(x[:n], exclusive=bool(ex), out_dtype=wide)
                line = []
                for v in [-1] + vs:
                    src, out = x[:n], o[:n]

                    def call():
                        if v < 0:
                            G.scan(src, exclusive=bool(ex), out=out, out_dtype=wide)
                        elif v >= 100:  # chunked: consecutive ring launches over 2^(v-100)-element slices (timing only)
                            ch = 1 << (v - 100)
                            for lo in range(0, n, ch):
                                m = min(ch, n - lo)
                                assert L.ring_ab_cfg(2, ex, DT[name], m, src[lo:].data_ptr(), out[lo:].data_ptr(),
                                                     ws.data_ptr(), s) == 0
                        else:
                            assert L.ring_ab_cfg(v, ex, DT[name], n, src.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                                 s) == 0
                    out.fill_(3)
                    call()
                    torch.cuda.synchronize()
                    ok = torch.equal(out, ref) or v >= 100
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
                    line.append(f"{'prod' if v < 0 else v}:{best:.1f}{'' if ok else '!FAIL'}")
                print(f"{name} 2^{lg} ex={ex}: " + "  ".join(line), flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:
        build()
    elif sys.argv[1] == "cfg":
        cfg()
    else:
        main()
