"""Time fp32 sum/dot variants (tuning lab, GPU only)."""
import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
LIB = os.path.join(HERE, os.environ.get("RED_LAB_LIB", "libred_lab.so"))
SRC = os.environ.get("RED_LAB_SRC", "red_lab.cu")


def build():
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared",
                           "-I", os.path.join(ROOT, "paper_1304_5553_b200", "csrc"), "-I", os.path.join(ROOT, "include"),
                           "-o", LIB, os.path.join(HERE, SRC)])


def main():
    import torch, synth
    from paper_1304_5553_b200 import gpuarray as G
    L = ctypes.CDLL(LIB)
    L.red_lab.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 5
    n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)
    dev = torch.device("cuda:0")
    x = synth.device_fill(synth.F32_U01, 1, n, device=dev)
    y = synth.device_fill(synth.F32_U01, 2, n, device=dev)
    out = torch.empty(1, device=dev)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    def t(fn, reps=30):
        for _ in range(3): fn()
        torch.cuda.synchronize(); e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    rs, rd = float(G.sum(x)), float(G.dot(x, y))
    ms = t(lambda: G.sum(x, out=out)); print(f"product sum {ms*1e3:7.1f} us {4*n/ms/1e6:7.1f} GB/s")
    ms = t(lambda: G.dot(x, y, out=out)); print(f"product dot {ms*1e3:7.1f} us {8*n/ms/1e6:7.1f} GB/s")
    ms = t(lambda: torch.sum(x)); print(f"torch sum   {ms*1e3:7.1f} us {4*n/ms/1e6:7.1f} GB/s")
    from paper_1304_5553_b200 import _abi
    wsr = G.workspace("reduce", x.device, s, _abi.gpuarray_reduce_workspace_bytes(0, n))
    args = (0, 0, 0, 0, n, x.data_ptr(), None, out.data_ptr(), wsr.data_ptr(), wsr.numel(), s)
    ms = t(lambda: _abi.LIB.gpuarray_reduce(*args)); print(f"raw-abi sum {ms*1e3:7.1f} us {4*n/ms/1e6:7.1f} GB/s")
    args = (0, 1, 0, 0, n, x.data_ptr(), y.data_ptr(), out.data_ptr(), wsr.data_ptr(), wsr.numel(), s)
    ms = t(lambda: _abi.LIB.gpuarray_reduce(*args)); print(f"raw-abi dot {ms*1e3:7.1f} us {8*n/ms/1e6:7.1f} GB/s")
    # step context: an axpbyz on other arrays right before each timed reduce
    z1 = torch.empty_like(x); x2 = torch.empty_like(x).fill_(1.0); y2 = torch.empty_like(x).fill_(2.0)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    def ctx(fn):
        for _ in range(3):
            G.axpbyz(5.0, x2, 6.0, y2, out=z1); fn()
        torch.cuda.synchronize()
        for a, b in ev:
            G.axpbyz(5.0, x2, 6.0, y2, out=z1)
            a.record(); fn(); b.record()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev) / len(ev)
    for name, fn, b in (("product sum", lambda: G.sum(x, out=out), 4), ("product dot", lambda: G.dot(x, y, out=out), 8)):
        ms = ctx(fn); print(f"ctx {name} {ms*1e3:7.1f} us {b*n/ms/1e6:7.1f} GB/s", flush=True)
    for v in (1, 11, 20, 21):
        b = 8 if v in (11, 21) else 4
        ms = ctx(lambda: L.red_lab(v, n, x.data_ptr(), y.data_ptr(), out.data_ptr(), ws.data_ptr(), s))
        print(f"ctx variant {v} {ms*1e3:7.1f} us {b*n/ms/1e6:7.1f} GB/s", flush=True)
    for v in ([int(q) for q in os.environ['RED_LAB_VARIANTS'].split(',')] if 'RED_LAB_VARIANTS' in os.environ else [1, 11]):
        dot = v in (10, 11, 12, 13, 14, 15, 16, 17, 21, 34, 35)
        L.red_lab(v, n, x.data_ptr(), y.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
        torch.cuda.synchronize()
        val = float(out[0])
        ok = abs(val - (rd if dot else rs)) <= 1e-5 * abs(rd if dot else rs)
        ms = t(lambda: L.red_lab(v, n, x.data_ptr(), y.data_ptr(), out.data_ptr(), ws.data_ptr(), s))
        b = 8 if dot else 4
        print(f"variant {v:3d} {'dot' if dot else 'sum'} {ms*1e3:7.1f} us {b*n/ms/1e6:7.1f} GB/s ok={ok}", flush=True)


if __name__ == "__main__":
    build() if sys.argv[1:2] == ["build"] else main()
