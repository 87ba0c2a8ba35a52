"""Reduction CTA shape at small / mid n (tuning lab, GPU only): variants of
red_shape_lab.cu timed cold (one call after an L2 flush) and warm (200 calls
replayed from a CUDA graph), fp32, n = 2^16 .. 2^24.
    RED_LAB_LIB=libred_shape.so RED_LAB_SRC=red_shape_lab.cu python tools/lab/run_red_lab.py build
    python tools/lab/run_red_small.py"""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1304_5553_b200 import gpuarray as G
    L = ctypes.CDLL(os.path.join(HERE, "libred_shape.so"))
    L.red_lab.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 5
    dev = torch.device("cuda:0")
    flush = torch.empty(512 * 2 ** 20 // 4, device=dev)
    clean = torch.ones(512 * 2 ** 20 // 4, device=dev)
    sink = torch.empty((), device=dev)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
    out = torch.empty(1, device=dev)
    st = torch.cuda.Stream(dev)
    variants = [int(v) for v in os.environ.get("VARIANTS", "5,3,8,9,15,13,18").split(",")]
    for lg in (16, 18, 20, 22, 24):
        n = 1 << lg
        x = torch.rand(n, device=dev)
        y = torch.rand(n, device=dev)
        line = []
        for v in variants:
            with torch.cuda.stream(st):
                s = st.cuda_stream
                fn = lambda: L.red_lab(v, n, x.data_ptr(), y.data_ptr(), out.data_ptr(), ws.data_ptr(), s)  # noqa
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                cold = []
                for _ in range(15):
                    flush.fill_(1.0)
                    G.sum(clean, out=sink)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    fn()
                    e1.record()
                    torch.cuda.synchronize()
                    cold.append(e0.elapsed_time(e1) * 1e3)
                cold.sort()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for _ in range(200):
                        fn()
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                warm = e0.elapsed_time(e1) * 1e3 / 200
            line.append(f"v{v}:{cold[7]:.1f}/{warm:.2f}")
        print(f"2^{lg} cold/warm us: " + "  ".join(line), flush=True)


if __name__ == "__main__":
    main()
