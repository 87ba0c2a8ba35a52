"""HBM-roofline sweep (BASELINE.json configs[1]: "HBM-roofline sweep over
n=2^16..2^30"): every hot-path op at n = 2^16 .. 2^30, timed with CUDA events
on the launching stream; when the working set is smaller than 4x L2 the L2 is
flushed before every timed call — a 512 MiB write, then a 512 MiB read of
another buffer so that the dirty lines of the write are written back before
the timed region (otherwise the op pays for them) — and only the op is timed.
Before every timed call the GPU is also given ~10 us of work (a device-side
sleep) so that the host enqueues the start event, the op and the stop event
while the stream is busy: the event interval then holds the op's device time,
not the host's launch latency (round 1's unflushed points, n >= 2^26 here,
included ~5 us of it).

    python tools/sweep.py [--min 16] [--max 30] [--reps 20] [--out gpurun_out/sweep.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1304_5553_b200 import gpuarray as G  # noqa: E402

L2_BYTES = 126 * 2 ** 20


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min", type=int, default=16)
    ap.add_argument("--max", type=int, default=30)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    clean = torch.ones(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    sink = torch.empty((), dtype=torch.float32, device=dev)
    pk = peak()
    rows = []
    ops = [
        ("axpbyz", torch.float32, 12), ("axpbyz", torch.float64, 24),
        ("norm2", torch.float32, 4), ("norm2", torch.float64, 8),
        ("dot", torch.float32, 8), ("sum", torch.float32, 4),
        ("scan", torch.int32, 8), ("scan", torch.int64, 16),
        ("scan_widen", torch.int32, 12),  # int32 in, int64 out (NEXT-2)
    ]
    for lg in range(a.min, a.max + 1):
        n = 1 << lg
        for name, dt, bpe in ops:
            esz = torch.tensor([], dtype=dt).element_size()
            need = 3 * n * esz if name in ("axpbyz", "scan_widen") else 2 * n * esz
            if need > torch.cuda.mem_get_info()[0] * 0.8:
                continue
            if dt.is_floating_point:
                kind = synth.F32_U01 if dt == torch.float32 else synth.F64_U01
                x = synth.device_fill(kind, 1, n, device=dev)
                y = synth.device_fill(kind, 2, n, device=dev)
            else:
                kind = synth.I32_RANGE if dt == torch.int32 else synth.I64_RANGE
                x = synth.device_fill(kind, 3, n, lo=0, hi=9, device=dev)
                y = None
            out = torch.empty(n, dtype=torch.int64, device=dev) if name == "scan_widen" else torch.empty_like(x)
            r = torch.empty((), dtype=dt, device=dev)
            fn = {
                "axpbyz": lambda: G.axpbyz(5.0, x, 6.0, y, out=out),
                "norm2": lambda: G.norm2sq(x, out=r),
                "dot": lambda: G.dot(x, y, out=r),
                "sum": lambda: G.sum(x, out=r),
                "scan": lambda: G.scan(x, exclusive=True, out=out),
                "scan_widen": lambda: G.scan(x, exclusive=True, out=out, out_dtype=torch.int64),
            }[name]
            small = need < 4 * L2_BYTES
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                if small:
                    flush.fill_(1.0)
                    G.sum(clean, out=sink)
                torch.cuda._sleep(20000)  # ~10 us of device time ahead of e0
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            med = ts[len(ts) // 2]
            gbs = n * bpe / (med * 1e-3) / 1e9
            rows.append({"op": name, "dtype": str(dt).replace("torch.", ""), "log2n": lg, "us_median": round(med * 1e3, 2),
                         "us_min": round(ts[0] * 1e3, 2), "gbs": round(gbs, 1), "frac_of_measured": round(gbs / pk, 4),
                         "frac_of_8tbs": round(gbs / 8000, 4), "l2_flushed": small})
            print(json.dumps(rows[-1]), flush=True)
            del x, y, out
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=0)


if __name__ == "__main__":
    main()
