"""Per-tile timeline of the single-touch scan (tuning lab, GPU only): one
traced call per variant at 2^28 int32 after warm-up, saved as .npy under
gpurun_out/ for tools/lab/trace_smem.py analyze.
    python tools/lab/trace_smem.py run | analyze"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
CASES = [(0, 0), (12, 296), (30, 0), (33, 296)]


def run():
    import torch
    L = ctypes.CDLL(os.path.join(HERE, "libsmem_lab.so"))
    L.smem_lab_trace.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    n = 1 << 28
    k = torch.randint(0, 10, (n,), dtype=torch.int32, device=dev)
    o = torch.empty_like(k)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
    tr = torch.zeros(8 * (n // 2048), dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for v, d in CASES:
        for _ in range(4):
            assert L.smem_lab_trace(v, n, k.data_ptr(), o.data_ptr(), ws.data_ptr(), d, tr.data_ptr(), s) == 0
        torch.cuda.synchronize()
        ntiles = n // (8 * (8192 if v in (0, 30) else 12288) // 4)
        np.save(os.path.join(ROOT, "gpurun_out", f"trace_smem_{v}.npy"), tr[: 8 * ntiles].view(-1, 8).cpu().numpy())


def analyze():
    for v, d in CASES:
        a = np.load(os.path.join(ROOT, "gpurun_out", f"trace_smem_{v}.npy")).astype(np.int64)
        t0 = a[:, 0].min()
        st, ld, ag, pf, en = [(a[:, i] - t0) / 1e3 for i in range(5)]
        ld = np.where(a[:, 1] > 0, ld, st)  # ragged tile has no stamp 1
        total = en.max()
        print(f"variant {v} (pf {d}): {len(a)} tiles, span {total:.1f} us")
        for name, x in (("load", ld - st), ("fold+publish", ag - ld), ("look-back", pf - ag), ("finish", en - pf),
                        ("life", en - st)):
            q = np.percentile(x[1:], [10, 50, 90, 99, 100])
            print(f"  {name:13s} mean {x[1:].mean():6.2f}  p10/50/90/99/max " + " ".join(f"{y:6.2f}" for y in q))
        # how far (in time) each tile's prefix lags its own aggregate, vs the latest predecessor aggregate
        lag = np.maximum.accumulate(ag) - ag
        print(f"  max-predecessor-aggregate lag: mean {lag.mean():.2f} p90 {np.percentile(lag, 90):.2f} us")
        # concurrency: tiles alive over time
        ts = np.linspace(0, total, 400)
        alive = [(st <= t).sum() - (en <= t).sum() for t in ts]
        print(f"  alive CTAs: median {np.median(alive):.0f} min(mid) {min(alive[40:-40]):.0f}")


if __name__ == "__main__":
    run() if sys.argv[1:] == ["run"] else analyze()
