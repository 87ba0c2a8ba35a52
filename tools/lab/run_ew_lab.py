"""Time fp32 axpbyz kernel variants (tuning lab, GPU only)."""
import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, "libew_lab.so")


def build():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared",
                           "-I", os.path.join(ROOT, "paper_1304_5553_b200", "csrc"), "-I", os.path.join(ROOT, "include"),
                           "-o", LIB, os.path.join(HERE, "ew_lab.cu")])


def main():
    import torch, synth
    from paper_1304_5553_b200 import gpuarray as G
    L = ctypes.CDLL(LIB)
    L.ew_lab.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)
    dev = torch.device("cuda:0")
    x = synth.device_fill(synth.F32_U01, 1, n, device=dev)
    y = synth.device_fill(synth.F32_U01, 2, n, device=dev)
    ref = G.axpbyz(5.0, x, -6.0, y)
    z = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    def t(fn, reps=30):
        for _ in range(3): fn()
        torch.cuda.synchronize(); e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    ms = t(lambda: G.axpbyz(5.0, x, -6.0, y, out=z))
    print(f"product        {ms*1e3:7.1f} us {12*n/ms/1e6:7.1f} GB/s", flush=True)
    ms = t(lambda: torch.add(x, y, alpha=2.0, out=z))
    print(f"torch.add      {ms*1e3:7.1f} us {12*n/ms/1e6:7.1f} GB/s", flush=True)
    for v in [0, 1, 2, 3, 4, 5, 6, 7, 10, 11, 12, 13, 14, 20, 21, 22, 23, 24, 25, 26, 27]:
        z.zero_()
        if L.ew_lab(v, n, 5.0, x.data_ptr(), -6.0, y.data_ptr(), z.data_ptr(), s) != 0:
            print("variant", v, "failed"); continue
        torch.cuda.synchronize()
        ok = torch.equal(z, ref)
        ms = t(lambda: L.ew_lab(v, n, 5.0, x.data_ptr(), -6.0, y.data_ptr(), z.data_ptr(), s))
        print(f"variant {v:3d}    {ms*1e3:7.1f} us {12*n/ms/1e6:7.1f} GB/s parity={'ok' if ok else 'FAIL'}", flush=True)


if __name__ == "__main__":
    build() if sys.argv[1:2] == ["build"] else main()
