"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/summarize_ncu.py <round-tag> <full.ncu-rep> [launches.csv]
    python tools/summarize_ncu.py traffic <log2n> <metrics.csv>

The second form reads an `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum
--csv` log of the bench's five hot-path launches at another size and records
their DRAM bytes per launch in profiles/ncu_traffic.json under <op>@2^<log2n>.

Writes profiles/<tag>_kernels.md (per-kernel metrics of the --set full
capture), profiles/<tag>_launches.md (share of each kernel in the launch
list of a bench run) and updates profiles/ncu_traffic.json (DRAM bytes per
launch of each hot-path kernel, read by bench.py's roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

OPS = ("axpbyz", "dot", "sum", "norm2", "scan")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
]


def op_of(name):
    if "ew_vec_kernel" in name:
        return "axpbyz" if ", true" in name or "1, 2" in name else "axpbz"
    if "reduce_kernel" in name:
        mp = name.split("reduce_kernel<")[1].split(">")[0].split(",")
        m = mp[3].strip()
        return {"0": "sum", "1": "dot", "2": "norm2"}.get(m, "reduce")
    if "scan" in name:
        return "scan"
    return name[:40]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_bytes(v, unit):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def traffic_from_metrics(log2n, path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    h = rows[0]
    ki, ni, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    ii = h.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        per[r[ii]][r[ni]] = to_bytes(r[vi].replace(",", ""), r[ui]) if "bytes" in r[ni] else r[vi]
        names[r[ii]] = r[ki]
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    seen = set()
    for i in sorted(per, key=int):
        op = op_of(names[i])
        if op in OPS and op not in seen:
            seen.add(op)
            traffic[f"{op}@2^{log2n}"] = int(per[i]["dram__bytes_read.sum"] + per[i]["dram__bytes_write.sum"])
            print(op, log2n, traffic[f"{op}@2^{log2n}"])
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)


def main():
    if sys.argv[1] == "traffic":
        return traffic_from_metrics(int(sys.argv[2]), sys.argv[3])
    tag, rep = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    os.makedirs(PROF, exist_ok=True)
    hdr, units, rows = raw_rows(rep)
    idx = {k: hdr.index(k) for k, _ in KEYS if k in hdr}
    lines = [f"# {tag}: ncu --set full --clock-control none (one launch per kernel, n = 2^28, `tools/profile_ops.py 28`)", "",
             "Source: `" + os.path.basename(rep) + "` (gpurun_out/, not committed). Durations are ncu's "
             "(serialised, cold-ish L2); compare shares, not absolutes, with bench.py.", "",
             "| op | kernel | " + " | ".join(n for _, n in KEYS) + " | DRAM GB/s |", "|" + "---|" * (len(KEYS) + 3)]
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        op = op_of(name)
        vals = []
        for k, _ in KEYS:
            vals.append(r[idx[k]] + " " + units[idx[k]] if k in idx else "-")
        rd = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
        wr = to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
        dur = float(r[idx["gpu__time_duration.sum"]]) * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}[units[idx["gpu__time_duration.sum"]]]
        lines.append(f"| {op} | `{name[:70]}` | " + " | ".join(vals) + f" | {(rd + wr) / dur / 1e9:.0f} |")
        traffic[f"{op}@2^28"] = int(rd + wr)
    open(os.path.join(PROF, f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    if launches:
        text = open(launches).read()
        start = text.find('"ID"')
        rows = list(csv.reader(io.StringIO(text[start:])))
        h = rows[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        # bench.py launches, in order: the input fills, W + K steps of the five
        # hot-path ops, then the e2e pipeline (2^24-element chunks).  The step
        # table keeps the first STEP_LAUNCHES launches of each op (3 warm-up +
        # 3 timed steps of `--steps 3 --warmup 3`); the e2e launches follow.
        STEP_LAUNCHES = 6
        tables = {"step": (defaultdict(float), defaultdict(int)), "all": (defaultdict(float), defaultdict(int))}
        for r in rows[1:]:
            if len(r) <= vi:
                continue
            v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1, "ms": 1e3}.get(r[ui], 1)
            op = op_of(r[ki])
            for name, (tot, cnt) in tables.items():
                if name == "step" and (op not in OPS or tables["step"][1][op] >= STEP_LAUNCHES):
                    continue
                tot[op] += v
                cnt[op] += 1
        out = [f"# {tag}: launch list of `bench.py --steps 3 --warmup 3` under "
               "`ncu --metrics gpu__time_duration.sum --clock-control none`", "",
               "Cold-cache, serialised per-launch times: the SHARE column of the step table is what must agree "
               "with bench.py's per-op split (ops.*.ms).", ""]
        for name, title in (("step", "Bench step (first 6 launches of each op: 3 warm-up + 3 timed steps, n = 2^33 per GPU)"),
                            ("all", "Every launch of the command (incl. the input fills and the e2e pipeline's "
                                    "2^24-element chunks)")):
            tot, cnt = tables[name]
            all_t = sum(tot.values())
            out += [f"## {title}", "", "| kernel (op) | launches | total us | mean us | share |", "|---|---|---|---|---|"]
            for op in sorted(tot, key=lambda o: -tot[o]):
                out.append(f"| {op} | {cnt[op]} | {tot[op]:.1f} | {tot[op] / cnt[op]:.1f} | {tot[op] / all_t * 100:.1f}% |")
            out.append("")
        open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(out))


if __name__ == "__main__":
    main()
