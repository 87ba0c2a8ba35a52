"""Attribute ncu warp-stall samples (SASS page csv) to CUDA source lines using
nvdisasm line info.  Usage: python tools/sass_lines.py <ncu_source.csv> <cubin> <mangled-function-substring>"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

csv_path, cubin, fn = sys.argv[1:4]
rows = list(csv.reader(open(csv_path)))
kname = rows[0][1] if rows and rows[0] and rows[0][0] == "Kernel Name" else ""
hdr = rows[1]
data = rows[2:]
i_a, i_s = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][i_a], 16)
samples = {int(r[i_a], 16) - base: float(r[i_s] or 0) for r in data}
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
reasons = {int(r[i_a], 16) - base: {hdr[i][6:]: float(r[i] or 0) for i in stall_cols} for r in data}
syms = subprocess.run(["cuobjdump", "-elf", cubin], capture_output=True, text=True).stdout
names = sorted(set(re.findall(r"(_Z\S*" + re.escape(fn) + r"\S*)", syms)))
name = names[0] if len(names) == 1 else None
if name is None:
    print("candidates:", names[:10])
    name = names[0]
full = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
start = full.find(".text." + name + ":")
end = full.find(".text.", start + 10)
dis = full[start:end if end > 0 else None]
line = None
per_line = defaultdict(float)
per_reason = defaultdict(lambda: defaultdict(float))
text = {}
for ln in dis.splitlines():
    m = re.search(r'line (\d+)', ln)
    if "//##" in ln and m:
        line = int(m.group(1))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*)", ln)
    if m:
        off = int(m.group(1), 16)
        if off in samples:
            per_line[line] += samples[off]
            for k, v in reasons[off].items():
                per_reason[line][k] += v
tot = sum(per_line.values()) or 1
for l, v in sorted(per_line.items(), key=lambda kv: -kv[1])[:25]:
    rs = sorted(per_reason[l].items(), key=lambda kv: -kv[1])[:3]
    print(f"{v / tot * 100:5.1f}%  line {l}  " + " ".join(f"{k}={x / (v or 1) * 100:.0f}%" for k, x in rs))
