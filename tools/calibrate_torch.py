"""Day-0 calibration with torch-only ops (no repo kernels): device query and
read-only / write-only / copy HBM ceilings, measured with CUDA events.
Writes gpurun_out/calib_torch.json. Measurement infrastructure only."""
import json, os, subprocess, time
import torch

def timeit(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return min(ts), sorted(ts)[len(ts) // 2]

out = {}
p = torch.cuda.get_device_properties(0)
out["device"] = {"name": p.name, "sms": p.multi_processor_count, "total_mem": p.total_memory,
                 "l2": getattr(p, "L2_cache_size", None)}
out["host"] = {"cores_affinity": len(os.sched_getaffinity(0)), "cpu_count": os.cpu_count()}
try:
    out["host"]["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
except Exception:
    pass
res = {}
for gib in (1, 4):
    n = gib * (1 << 30) // 4
    a = torch.empty(n, dtype=torch.float32, device="cuda").uniform_()
    b = torch.empty_like(a)
    tmin, tmed = timeit(lambda: b.copy_(a))
    res[f"copy_{gib}GiB"] = 2 * n * 4 / tmin / 1e9
    tmin, tmed = timeit(lambda: b.fill_(1.0))
    res[f"fill_{gib}GiB"] = n * 4 / tmin / 1e9
    tmin, tmed = timeit(lambda: a.sum())
    res[f"sum_{gib}GiB"] = n * 4 / tmin / 1e9
    c = torch.empty_like(a)
    tmin, tmed = timeit(lambda: torch.add(a, b, alpha=2.0, out=c))
    res[f"add_{gib}GiB"] = 3 * n * 4 / tmin / 1e9
    del a, b, c
    torch.cuda.empty_cache()
out["torch_gbs"] = res
out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,clocks.max.mem,power.limit", "--format=csv"], capture_output=True, text=True).stdout
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/calib_torch.json", "w"), indent=1)
print(json.dumps(out, indent=1))
