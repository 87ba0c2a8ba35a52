"""Render tools/sweep.py output as the committed markdown table.
    python tools/sweep_table.py gpurun_out/sweep.json profiles/r1_sweep.md"""
import json
import sys

rows = json.load(open(sys.argv[1]))
ops = sorted({(r["op"], r["dtype"]) for r in rows})
lgs = sorted({r["log2n"] for r in rows})
d = {(r["op"], r["dtype"], r["log2n"]): r for r in rows}
out = ["# HBM-roofline sweep, n = 2^16 .. 2^30 (one B200)", "",
       "`python tools/sweep.py`: median of 15 CUDA-event-timed calls per point; working sets below 4x L2 are "
       "flushed (512 MiB write, then a 512 MiB read of another buffer) before every call, and a ~10 us device sleep "
       "precedes every timed call so the events measure device time, not host launch latency.  Algorithmic GB/s "
       "(axpbyz 12/24 B, dot 8, sum/norm2 4/8, scan 8/16 B per element).  Small n is launch- and "
       "latency-bound (a 2^16 fp32 sum is 256 KiB).", "",
       "| op | dtype | " + " | ".join(f"2^{l}" for l in lgs) + " |", "|---|---|" + "---|" * len(lgs)]
for op, dt in ops:
    out.append(f"| {op} | {dt} | " + " | ".join(f"{d[(op, dt, l)]['gbs']:.0f}" if (op, dt, l) in d else "-"
                                              for l in lgs) + " |")
out += ["", "Fraction of the measured copy peak (MEASURED_PEAKS.json hbm_gbs) at the BASELINE sizes:", "",
        "| op | dtype | 2^26 (256 MiB fp32) | 2^28 | 2^30 |", "|---|---|---|---|---|"]
for op, dt in ops:
    cells = []
    for l in (26, 28, 30):
        r = d.get((op, dt, l))
        cells.append(f"{r['frac_of_measured']:.3f} ({r['frac_of_8tbs']:.3f} of 8 TB/s)" if r else "-")
    out.append(f"| {op} | {dt} | " + " | ".join(cells) + " |")
open(sys.argv[2], "w").write("\n".join(out) + "\n")
