"""Widened int32 -> int64 exclusive scan, 512-byte vs 1 KiB rows (tuning lab,
GPU only): tile_lab.cu lab_scan_wide variants, back-to-back calls, parity
against the product.   python tools/lab/run_wide_lab.py [lo hi]"""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1304_5553_b200 import gpuarray as G
    L = ctypes.CDLL(os.path.join(HERE, "libtile_lab.so"))
    L.lab_scan_wide.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 4
    lo, hi = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (26, 30)
    dev = torch.device("cuda:0")
    k = torch.randint(0, 10, (1 << hi,), dtype=torch.int32, device=dev)
    o = torch.empty(1 << hi, dtype=torch.int64, device=dev)
    ws = torch.zeros(1 << 24, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for lg in range(lo, hi + 1):
        n = 1 << lg
        line = []
        for v in (0, 1, 2, 3, 0):
            ws.zero_()
            assert L.lab_scan_wide(v, n, k.data_ptr(), o.data_ptr(), ws.data_ptr(), s) == 0
            torch.cuda.synchronize()
            ok = torch.equal(o[:n], G.scan(k[:n], exclusive=True, out_dtype=torch.int64))
            best = 1e30
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    L.lab_scan_wide(v, n, k.data_ptr(), o.data_ptr(), ws.data_ptr(), s)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / 5 * 1e3)
            line.append(f"{v}:{best:.1f}us{'' if ok else '!FAIL'}")
        print(f"2^{lg}: " + "  ".join(line), flush=True)


if __name__ == "__main__":
    main()
