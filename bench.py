"""bench.py — throughput of the GPUArray hot path on B200 (BASELINE.json metric:
"achieved HBM GB/s (and % of 8 TB/s peak) for dot/sum/axpbyz/scan at 1/2/4/8 B200").

Default workload: the BASELINE metric grid — ONE global
array of n_global = 2^33 elements, sharded contiguously over the N ranks
(strong scaling: the same global arrays at every N; shard g holds global
indices [floor(g n/N), floor((g+1) n/N)) of the counter-based generator,
DESIGN.md R16/R20).  One STEP = one pass of every hot-path row (§8(a)) over
the global arrays:
    z = axpbyz(5, x, 6, y)           fp32, 12 B/elt      (a1)
    dot(x, y), sum(x), norm2sq(x)    fp32, 8/4/4 B/elt   (a2-a4; + a6 NCCL allreduce at N>1: C4)
    exclusive scan(k)                int32, 8 B/elt      (a5; + a7 totals allgather + carry at N>1: C5)
x, y ~ U[0,1) fp32, k ~ U{0..9} int32; at N = 1 that is 4 arrays of 32 GiB
(z and the scan output share one buffer; 128 GiB of HBM), far larger than
the 126 MB L2, so no flush is needed between steps.

value = algorithmic bytes of the global step / max-over-ranks device time.

Extras on the same line (N = 1 only; BASELINE.json single-GPU configs):
    c3       int32 / int64 sum, max and inclusive scan at n = 2^30
    c2_fp64  fp64 axpbyz and squared 2-norm at n = 2^28
each op timed alone (CUDA events, R reps), with a sampled parity check.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (driver, N > 1)

--impl reference times the CPU oracle (oracle/, test infrastructure) on the
host cores on a bounded sample of the same workload: there is no reference
implementation to install (the paper ships no code).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LOG2_N_GLOBAL = 33
A, B = 5.0, 6.0
# algorithmic bytes per element
OP_BYTES = {"axpbyz": 12, "dot": 8, "sum": 4, "norm2": 4, "scan": 8}
OPS = list(OP_BYTES)
PEAK_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
NOMINAL_GBS = 8000.0
METRIC = "achieved HBM GB/s (and % of 8 TB/s peak) for dot/sum/axpbyz/scan at 1/2/4/8 B200"
WORKLOAD = ("BASELINE metric grid (configs[3]/[4] generators): axpbyz(5,x,6,y) + dot + sum + norm2 fp32 U[0,1) "
            "and exclusive scan int32 U{0..9} over ONE global array of n_global elements sharded contiguously "
            "over the GPUs (strong scaling)")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--log2n-global", type=int, default=LOG2_N_GLOBAL,
                   help="global elements per array = 2^k (default 33, the BASELINE metric grid)")
    p.add_argument("--e2e-log2n", type=int, default=28, help="elements per rank of the end-to-end slice = 2^k")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the c3 / c2_fp64 blocks")
    p.add_argument("--collective", choices=["nccl", "fused"], default="nccl",
                   help="N>1: the C entries gpuarray_reduce_sharded / gpuarray_scan_sharded with NCCL (default), or "
                        "the fused in-kernel NVLink finish (gpuarray_reduce_xgpu over torch symmetric memory)")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy_ 1 Gi bf16)"
    except Exception:
        return PEAK_FALLBACK_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 100 ms while the timed region runs."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [q.strip() for q in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle leg
class OracleStep:
    """The oracle (as it stands, single-threaded plain C) on a bounded sample
    of the workload: the same five ops on 2^log2m elements regenerated once
    by the synth host twin.  Only the compute is timed."""

    def __init__(self, log2m):
        import oracle
        import synth
        self.oracle = oracle
        self.m = 1 << log2m
        self.log2m = log2m
        self.x = synth.host_fill(synth.F32_U01, synth.SEED_X, self.m)
        self.y = synth.host_fill(synth.F32_U01, synth.SEED_Y, self.m)
        self.k = synth.host_fill(synth.I32_RANGE, synth.SEED_INT, self.m, lo=0, hi=9)

    def __call__(self):
        import numpy as np
        o = self.oracle
        t0 = time.perf_counter()
        o.axpbyz(np.float32(A), self.x, np.float32(B), self.y)
        o.reduce(o.SUM, o.MAP_MUL, self.x, self.y)
        o.reduce(o.SUM, o.MAP_ID, self.x)
        o.reduce(o.SUM, o.MAP_SQUARE, self.x)
        o.scan(o.EXCLUSIVE, self.k)
        return time.perf_counter() - t0

    @property
    def bytes(self):
        return self.m * sum(OP_BYTES.values())

    def describe(self):
        return (f"2^{self.log2m} elements per op (axpbyz/dot/sum/norm2 fp32 + exclusive scan int32) of the same "
                f"synthetic streams (global indices [0, 2^{self.log2m})), regenerated once by the synth host twin; "
                f"oracle compute only; 1 thread (plain single-threaded C, -O2 -ffp-contract=off)")


def oracle_sample(log2m, min_seconds=10.0, min_reps=3):
    """The oracle over the 2^log2m sample, repeated until at least
    min_seconds of CPU compute have been timed (the bounded 10-30 s sample
    the contract asks for); GB/s = all bytes / all timed seconds."""
    step = OracleStep(log2m)
    step()
    secs, reps = 0.0, 0
    while reps < min_reps or secs < min_seconds:
        secs += step()
        reps += 1
    desc = step.describe() + f"; the sample repeated {reps} times ({secs:.1f} s of oracle compute timed)"
    return step.bytes * reps / secs / 1e9, secs, desc


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle on the host cores (rank 0 only; the
    paper ships no code, so the oracle is the reference arm)."""
    if rank != 0:
        return
    step = OracleStep(min(args.log2n_global, 24))
    for _ in range(max(args.warmup, 1)):
        step()
    times = [step() for _ in range(max(args.steps, 1))]
    total = sum(times)
    gbs = step.bytes * len(times) / total / 1e9
    n_full = 1 << args.log2n_global
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world,
        "steps": len(times), "warmup": max(args.warmup, 1), "ms_per_step": round(total / len(times) * 1e3, 3),
        "ms_per_full_step_extrapolated": round(n_full * sum(OP_BYTES.values()) / (gbs * 1e9) * 1e3, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+i32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_global": n_full,
                   "sample": f"each reference step is a 2^{step.log2m}-element sample of the 2^{args.log2n_global} "
                             f"global arrays", "parallelism": "cpu, 1 thread"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": step.describe()},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "no reference code exists (the paper ships none, BASELINE.json published = {}); the reference "
                "arm is the CPU oracle timed on a bounded sample of the same workload",
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ sampled parity
def windows(n, count=8, width=4096):
    """`count` index windows [a, a+width) spread over [0, n), always including
    the first and the last elements."""
    if n <= width:
        return [(0, n)] if n else []
    starts = sorted({0, n - width, *[(n - width) * j // (count - 1) for j in range(count)]})
    return [(a, a + width) for a in starts]


def lib_prefix_i64(torch, k, a, chunk=1 << 26):
    """sum(k[:a]) as a Python int, from torch's int64 sums of <= 2^26-element
    slices (a library result, independent of our kernels; bounded memory)."""
    return sum(int(k[lo:min(a, lo + chunk)].sum(dtype=torch.int64).item()) for lo in range(0, a, chunk))


def lib_sums_f64(torch, x, y, chunk=1 << 26):
    """torch float64 (dot(x, y), sum(x), sum(x*x)) over <= 2^26-element
    slices: the library check of the reductions (bounded memory)."""
    acc = torch.zeros(3, dtype=torch.float64, device=x.device)
    for lo in range(0, x.numel(), chunk):
        xd = x[lo:lo + chunk].double()
        acc += torch.stack([(xd * y[lo:lo + chunk].double()).sum(), xd.sum(), (xd * xd).sum()])
    return acc


def parity_main(torch, G, x, y, k, z, s, start, cnt, rank, world, exchange=None, gdist=None, dist=None):
    """Untimed pass of the step after the timed loop, checked against the CPU
    oracle on sampled windows (axpbyz bit-exact; scan bit-exact, each
    window's carry-in from torch's int64 sum of everything before it, a
    library result independent of our kernels) and the reductions against
    torch's float64 reductions of the same shard (a library check; full
    oracle parity at these sizes lives in tests/)."""
    import numpy as np

    import oracle
    import synth
    details, ok = {}, True
    G.axpbyz(A, x, B, y, out=z)
    bad = 0
    for a, b in windows(cnt):
        xh = synth.host_fill(synth.F32_U01, synth.SEED_X, b - a, start=start + a)
        yh = synth.host_fill(synth.F32_U01, synth.SEED_Y, b - a, start=start + a)
        want = oracle.axpbyz(np.float32(A), xh, np.float32(B), yh).view(np.uint32)
        bad += int((z[a:b].cpu().numpy().view(np.uint32) != want).sum())
    details["axpbyz_window_mismatches"] = bad
    ok &= bad == 0
    if exchange is not None:
        red = [gdist.reduce_fused(G.SUM, m, x, y if m == G.MUL else None, exchange=exchange) for m in (G.MUL, G.ID,
                                                                                                       G.SQUARE)]
    elif world > 1:
        red = [gdist.reduce(G.SUM, m, x, y if m == G.MUL else None) for m in (G.MUL, G.ID, G.SQUARE)]
    else:
        red = [G.reduce(G.SUM, m, x, y if m == G.MUL else None) for m in (G.MUL, G.ID, G.SQUARE)]
    lib = lib_sums_f64(torch, x, y)
    if world > 1:
        dist.all_reduce(lib)
    rel = [abs(float(r.item()) - float(v)) / abs(float(v)) for r, v in zip(red, lib.tolist())]
    details["reduction_rel_err_vs_torch_f64"] = [float(f"{e:.3g}") for e in rel]
    ok &= all(e <= 1e-5 for e in rel)
    if exchange is not None:
        gdist.scan_fused(k, exclusive=True, out=s, exchange=exchange)
    elif world > 1:
        gdist.scan(k, exclusive=True, out=s)
    else:
        G.scan(k, exclusive=True, out=s)
    # global exclusive prefix in front of each window: earlier ranks' totals
    # plus this shard's prefix (torch int64 sums, wrapped to int32)
    tot = torch.tensor([lib_prefix_i64(torch, k, cnt)], dtype=torch.int64, device=k.device)
    if world > 1:
        alltot = torch.empty(world, dtype=torch.int64, device=k.device)
        dist.all_gather_into_tensor(alltot, tot)
        before = int(alltot[:rank].sum().item())
    else:
        before = 0
    bad = 0
    for a, b in windows(cnt):
        kh = synth.host_fill(synth.I32_RANGE, synth.SEED_INT, b - a, start=start + a, lo=0, hi=9)
        c = (before + lib_prefix_i64(torch, k, a)) & 0xffffffff
        c = c - (1 << 32) if c >= 1 << 31 else c
        want = oracle.scan(oracle.EXCLUSIVE, kh, carry=np.int32(c))
        bad += int((s[a:b].cpu().numpy() != want).sum())
    details["scan_window_mismatches"] = bad
    ok &= bad == 0
    details["windows"] = f"{len(windows(cnt))} x 4096 elements per rank (first, last, spread)"
    return ok, details


# ------------------------------------------------------------------ extras (N = 1)
def time_op(torch, fn, reps):
    fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return statistics.median(ts), ts[0]


def run_extras(torch, G, dev, reps=10):
    """configs[2] (C3) and the fp64 half of configs[1] (C2), each op timed
    alone, with sampled parity (bit-exact integer results against torch's
    library reductions; scan windows against the oracle)."""
    import numpy as np

    import oracle
    import synth
    out = {}

    def entry(name, n, bpe, fn, ok):
        med, best = time_op(torch, fn, reps)
        gbs = n * bpe / (med * 1e-3) / 1e9
        out[name] = {"n": n, "ms": round(med, 4), "ms_min": round(best, 4), "gbs": round(gbs, 1),
                     "frac_of_8tbs": round(gbs / NOMINAL_GBS, 4), "bytes_per_elt": bpe, "parity": bool(ok)}

    n = 1 << 30
    for dt, kind, tdt in ((np.int32, synth.I32_RANGE, torch.int32), (np.int64, synth.I64_RANGE, torch.int64)):
        sz = np.dtype(dt).itemsize
        tag = "i32" if dt == np.int32 else "i64"
        kk = synth.device_fill(kind, synth.SEED_INT, n, lo=0, hi=9, device=dev)
        r = torch.empty((), dtype=tdt, device=dev)
        G.sum(kk, out=r)
        ok = int(r.item()) == lib_prefix_i64(torch, kk, n)  # no wrap in int64 (9 * 2^30 < 2^63)
        if dt == np.int32:  # int32 wraps: compare modulo 2^32
            ok = (int(r.item()) & 0xffffffff) == (lib_prefix_i64(torch, kk, n) & 0xffffffff)
        entry(f"sum_{tag}", n, sz, lambda: G.sum(kk, out=r), ok)
        mx = synth.device_fill(kind, synth.SEED_MAXMIN, n, lo=-(1 << 31), hi=(1 << 31) - 1, device=dev)
        mx[n // 3] = np.iinfo(dt).max  # a planted extreme (C3)
        G.max(mx, out=r)
        entry(f"max_{tag}", n, sz, lambda: G.max(mx, out=r), int(r.item()) == int(mx.max().item()))
        del mx
        sc = torch.empty_like(kk)
        G.scan(kk, out=sc)
        bad = 0
        for a, b in windows(n):
            kh = synth.host_fill(kind, synth.SEED_INT, b - a, start=a, lo=0, hi=9)
            c = lib_prefix_i64(torch, kk, a)
            if dt == np.int32:
                c &= 0xffffffff
                c = c - (1 << 32) if c >= 1 << 31 else c
            want = oracle.scan(oracle.INCLUSIVE, kh, carry=dt(c))
            bad += int((sc[a:b].cpu().numpy() != want).sum())
        entry(f"scan_incl_{tag}", n, 2 * sz, lambda: G.scan(kk, out=sc), bad == 0)
        del kk, sc
        torch.cuda.empty_cache()
    n = 1 << 28
    x = synth.device_fill(synth.F64_U01, synth.SEED_X, n, device=dev)
    y = synth.device_fill(synth.F64_U01, synth.SEED_Y, n, device=dev)
    z = torch.empty_like(x)
    G.axpbyz(A, x, B, y, out=z)
    bad = 0
    for a, b in windows(n):
        xh = synth.host_fill(synth.F64_U01, synth.SEED_X, b - a, start=a)
        yh = synth.host_fill(synth.F64_U01, synth.SEED_Y, b - a, start=a)
        bad += int((z[a:b].cpu().numpy().view(np.uint64) != oracle.axpbyz(np.float64(A), xh, np.float64(B),
                                                                          yh).view(np.uint64)).sum())
    entry("axpbyz_f64", n, 24, lambda: G.axpbyz(A, x, B, y, out=z), bad == 0)
    r = torch.empty((), dtype=torch.float64, device=dev)
    G.norm2sq(x, out=r)
    ref = float(lib_sums_f64(torch, x, x)[2].item())
    entry("norm2_f64", n, 8, lambda: G.norm2sq(x, out=r), abs(float(r.item()) - ref) <= 1e-12 * abs(ref))
    del x, y, z
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ GPU leg
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    import synth
    import paper_1304_5553_b200 as ga
    from paper_1304_5553_b200 import dist as gdist
    from paper_1304_5553_b200 import gpuarray as G

    # BENCH_SHARE_GPU=1 (testing only): every rank uses cuda:0 and gloo, so the
    # N > 1 choreography can be exercised on a one-GPU box; numbers from such a
    # run are not bench values.
    share = os.environ.get("BENCH_SHARE_GPU") == "1"
    dev_index = 0 if share else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    n_global = 1 << args.log2n_global
    start, cnt = gdist.shard_range(n_global, world, rank)
    x = synth.device_fill(synth.F32_U01, synth.SEED_X, cnt, start=start, device=dev)
    y = synth.device_fill(synth.F32_U01, synth.SEED_Y, cnt, start=start, device=dev)
    k = synth.device_fill(synth.I32_RANGE, synth.SEED_INT, cnt, start=start, lo=0, hi=9, device=dev)
    z = torch.empty_like(x)
    s = z.view(torch.int32)  # the scan output shares z's buffer (HBM budget at n = 2^33 on one GPU)
    red = torch.empty(3, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    ev = {op: [] for op in OPS}
    xch = None
    if world > 1 and args.collective == "fused":
        xch = gdist.Exchange.symmetric(device=dev)
        offset = torch.empty(1, dtype=torch.int32, device=dev)

    def step(record):
        def mark():
            if record:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                return e
            return None
        e0 = mark()
        G.axpbyz(A, x, B, y, out=z)
        e1 = mark()
        if xch is not None:  # fused: each reduction finishes across GPUs inside its own kernel
            gdist.reduce_fused(G.SUM, G.MUL, x, y, out=red[0:1], exchange=xch)
            e2 = mark()
            gdist.reduce_fused(G.SUM, G.ID, x, out=red[1:2], exchange=xch)
            e3 = mark()
            gdist.reduce_fused(G.SUM, G.SQUARE, x, out=red[2:3], exchange=xch)
            e4 = mark()
            gdist.scan_fused(k, exclusive=True, out=s, exchange=xch, offset=offset)
        else:  # world == 1: the local kernels; world > 1: + NCCL inside the C entries
            gdist.reduce(G.SUM, G.MUL, x, y, out=red[0:1])
            e2 = mark()
            gdist.reduce(G.SUM, G.ID, x, out=red[1:2])
            e3 = mark()
            gdist.reduce(G.SUM, G.SQUARE, x, out=red[2:3])
            e4 = mark()
            gdist.scan(k, exclusive=True, out=s)
        e5 = mark()
        if record:
            for op, (a, b) in zip(OPS, ((e0, e1), (e1, e2), (e2, e3), (e3, e4), (e4, e5))):
                ev[op].append((a, b))

    for _ in range(max(args.warmup, 3)):
        step(False)
    torch.cuda.synchronize()

    clocks = ClockSampler(dev_index)
    clocks.start()
    time.sleep(0.3)  # let the sampler start
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ga.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_stop = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for _ in range(args.steps):
        step(True)
    t_stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ga.launch_count() - launches0
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_stop)

    per_op_ms = {op: sum(a.elapsed_time(b) for a, b in ev[op]) / len(ev[op]) for op in OPS}
    t = torch.tensor([elapsed_ms] + [per_op_ms[op] for op in OPS], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t[0])
    per_op_ms = {op: float(v) for op, v in zip(OPS, t[1:].tolist())}

    # ---- parity of this run's step (untimed pass, sampled; full parity is in tests/)
    par_ok, par = parity_main(torch, G, x, y, k, z, s, start, cnt, rank, world, exchange=xch, gdist=gdist,
                              dist=dist)
    if world > 1:
        flag = torch.tensor([0 if par_ok else 1], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        par_ok = int(flag.item()) == 0
    del x, y, k, z, s
    torch.cuda.empty_cache()

    # ---- end-to-end through the public API with host buffers (bounded slice)
    e2e = run_e2e(args, world, rank, dev, ga, G, gdist, torch, dist)
    extras = None
    if world == 1 and not args.no_extras:
        extras = run_extras(torch, G, dev)

    if rank == 0:
        peak, peak_src = peaks()
        step_bytes = n_global * sum(OP_BYTES.values())
        ms_per_step = elapsed_ms / args.steps
        value = step_bytes / (ms_per_step * 1e-3) / 1e9
        ops = {}
        for op in OPS:
            gbs = n_global * OP_BYTES[op] / (per_op_ms[op] * 1e-3) / 1e9
            ops[op] = {"ms": round(per_op_ms[op], 4), "gbs": round(gbs, 1),
                       "frac_of_measured": round(gbs / world / peak, 4),
                       "frac_of_8tbs": round(gbs / world / NOMINAL_GBS, 4), "bytes_per_elt": OP_BYTES[op]}
        if world > 1:
            ops["scan"]["note"] = ("per element the sharded scan reads the shard twice (reduce, then scan with "
                                   "carry) and writes it once: implementation floor 12 B/elt (DESIGN.md R18); gbs "
                                   "counts the 8 algorithmic B/elt")
        dom = max(OPS, key=lambda o: per_op_ms[o])
        ach = cnt * OP_BYTES[dom] / (per_op_ms[dom] * 1e-3) / 1e9  # per GPU, per launch
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "peak_source": peak_src,
                "traffic": ncu_traffic(dom, args.log2n_global - (world.bit_length() - 1)),
                "algorithmic_bytes_per_launch": cnt * OP_BYTES[dom],
                "unit_of_work": f"{OP_BYTES[dom]} B per element x {cnt} elements per launch (one GPU's shard)"}
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            g, secs, desc = oracle_sample(24)
            cpu = {"value": round(g, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": desc,
                   "seconds": round(secs, 3)}
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+i32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_global": n_global, "log2n_global": args.log2n_global,
                       "n_per_gpu": cnt, "parallelism": f"dp{world} (contiguous shards)",
                       "buffers": "x, y fp32, k int32, z fp32 (also the scan output) per GPU",
                       "l2": ("arrays >= 1 GiB per GPU, > 126 MB L2: no flush needed" if cnt >= 1 << 28 else
                              "arrays smaller than 4x L2: L2-warm numbers")},
            "frac_of_8tbs": round(value / world / NOMINAL_GBS, 4),
            "elements_per_s": round(n_global * len(OPS) / (ms_per_step * 1e-3), 1),
            "ops": ops, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "parity": {"ok": bool(par_ok), **par},
            "gpu_launches": int(launches), "launches_per_step": launches / args.steps, "clocks": clk,
            "collective": ("none (single GPU)" if world == 1 else
                           "fused in-kernel NVLink finish" if xch is not None else
                           "gloo via torch.distributed (BENCH_SHARE_GPU test mode: ranks share one GPU)" if share else
                           "NCCL inside gpuarray_reduce_sharded / gpuarray_scan_sharded"),
        }
        if extras is not None:
            line["extras"] = extras
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, world, rank, dev, ga, G, gdist, torch, dist):
    """The same step through the public API with pinned HOST inputs, on a
    bounded slice of 2^e2e_log2n elements per rank (global indices
    [rank*m, (rank+1)*m)): H2D of x, y, k, the five ops, D2H of z, the scan
    output and the three scalars — all inside the timed region.  The step is
    pipelined over chunks of 2^24 elements on three streams (H2D of chunk c+1
    || compute of chunk c || D2H of chunk c-1; PCIe is full duplex), so the
    host link, not the HBM, bounds it.  Chunk results are combined with the
    same kernels: per-chunk reduction partials are folded by one more
    reduction, and each chunk's scan takes the sums of the earlier chunks
    (and, at N > 1, of the earlier ranks) as carry-in."""
    import synth
    steps = max(1, args.e2e_steps)
    n = 1 << args.e2e_log2n
    start = rank * n
    xh = torch.empty(n, dtype=torch.float32, pin_memory=True)
    yh = torch.empty(n, dtype=torch.float32, pin_memory=True)
    kh = torch.empty(n, dtype=torch.int32, pin_memory=True)
    synth.host_fill(synth.F32_U01, synth.SEED_X, n, start=start, out=xh.numpy())
    synth.host_fill(synth.F32_U01, synth.SEED_Y, n, start=start, out=yh.numpy())
    synth.host_fill(synth.I32_RANGE, synth.SEED_INT, n, start=start, lo=0, hi=9, out=kh.numpy())
    zh = torch.empty(n, dtype=torch.float32, pin_memory=True)
    sh = torch.empty(n, dtype=torch.int32, pin_memory=True)
    rh = torch.empty(3, dtype=torch.float32, pin_memory=True)

    chunk = min(n, 1 << 24)
    nch = (n + chunk - 1) // chunk
    slots = 3
    s_in, s_cmp, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    xd = [torch.empty(chunk, dtype=torch.float32, device=dev) for _ in range(slots)]
    yd = [torch.empty(chunk, dtype=torch.float32, device=dev) for _ in range(slots)]
    kd = [torch.empty(chunk, dtype=torch.int32, device=dev) for _ in range(slots)]
    zd = [torch.empty(chunk, dtype=torch.float32, device=dev) for _ in range(slots)]
    sd = [torch.empty(chunk, dtype=torch.int32, device=dev) for _ in range(slots)]
    part = torch.empty(3, nch, dtype=torch.float32, device=dev)   # per-chunk dot / sum / norm2
    ksum = torch.empty(nch + 1, dtype=torch.int32, device=dev)    # [0]: offset of this rank, then chunk sums
    red = torch.empty(3, dtype=torch.float32, device=dev)
    totals = torch.empty(world + 1, dtype=torch.int32, device=dev)

    kfull = torch.empty(n, dtype=torch.int32, device=dev) if world > 1 else None

    def one():
        ev_in = [torch.cuda.Event() for _ in range(nch)]
        ev_cmp = [torch.cuda.Event() for _ in range(nch)]
        ev_out = [torch.cuda.Event() for _ in range(nch)]
        if world > 1:
            # The scan offset of this rank needs the totals of the earlier
            # ranks before any chunk can be finished: k comes over whole,
            # first, and its total is exchanged (one all_gather).
            with torch.cuda.stream(s_cmp):
                kfull.copy_(kh, non_blocking=True)
                mine = totals[world:]
                G.reduce(G.SUM, G.ID, kfull, out=mine)
                dist.all_gather_into_tensor(totals[:world], mine)
                r = dist.get_rank()
                if r > 0:
                    G.reduce(G.SUM, G.ID, totals[:r], out=ksum[0:1])
                else:
                    ksum[0:1].zero_()
        else:
            with torch.cuda.stream(s_cmp):
                ksum[0:1].zero_()
        for c in range(nch):
            sl, lo, hi = c % slots, c * chunk, min(n, (c + 1) * chunk)
            m = hi - lo
            with torch.cuda.stream(s_in):
                if c >= slots:
                    s_in.wait_event(ev_out[c - slots])  # slot's previous results copied out
                xd[sl][:m].copy_(xh[lo:hi], non_blocking=True)
                yd[sl][:m].copy_(yh[lo:hi], non_blocking=True)
                if world == 1:
                    kd[sl][:m].copy_(kh[lo:hi], non_blocking=True)
                ev_in[c].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[c])
                x, y = xd[sl][:m], yd[sl][:m]
                k = kd[sl][:m] if world == 1 else kfull[lo:hi]
                G.axpbyz(A, x, B, y, out=zd[sl][:m])
                G.reduce(G.SUM, G.MUL, x, y, out=part[0, c:c + 1])
                G.reduce(G.SUM, G.ID, x, out=part[1, c:c + 1])
                G.reduce(G.SUM, G.SQUARE, x, out=part[2, c:c + 1])
                G.reduce(G.SUM, G.ID, k, out=ksum[c + 1:c + 2])
                G.scan(k, exclusive=True, out=sd[sl][:m], carry=ksum[:c + 1])
                ev_cmp[c].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[c])
                zh[lo:hi].copy_(zd[sl][:m], non_blocking=True)
                sh[lo:hi].copy_(sd[sl][:m], non_blocking=True)
                ev_out[c].record(s_out)
        with torch.cuda.stream(s_cmp):
            for q in range(3):
                G.reduce(G.SUM, G.ID, part[q], out=red[q:q + 1])
            if world > 1:
                dist.all_reduce(red, op=dist.ReduceOp.SUM)
            rh.copy_(red, non_blocking=True)
        torch.cuda.synchronize(dev)
        return float(rh[0])

    one()
    # spot check of the pipelined results (full parity lives in tests/):
    # sampled z against the oracle, the scan's head against the oracle
    import numpy as np

    import oracle
    idx = np.arange(0, n, max(1, n // 4096))
    zx = oracle.axpbyz(np.float32(A), xh.numpy()[idx], np.float32(B), yh.numpy()[idx])
    e2e_check = bool(np.array_equal(zh.numpy()[idx].view(np.uint32), zx.view(np.uint32)))
    if world == 1:
        m = min(n, 1 << 20)
        e2e_check = e2e_check and bool(np.array_equal(sh.numpy()[:m], oracle.scan(oracle.EXCLUSIVE, kh.numpy()[:m])))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        one()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    tt = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt[0])
    step_bytes = n * sum(OP_BYTES.values())
    res = {"value": round(world * step_bytes / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": 3 * n * 4, "d2h_bytes_per_step": 2 * n * 4 + 3 * 4, "ms_per_step": round(ms, 3),
           "steps": steps, "n_per_gpu": n, "chunk_elements": chunk, "e2e_parity": e2e_check,
           "path": "pinned host -> device copies + paper_1304_5553_b200 public API + device -> host, "
                   "pipelined over 2^24-element chunks on three streams",
           "slice": f"bounded slice: 2^{args.e2e_log2n} elements per GPU (global indices [rank*2^{args.e2e_log2n}, "
                    f"(rank+1)*2^{args.e2e_log2n})); the host link, not HBM, bounds it"}
    del xh, yh, kh, zh, sh
    return res


def ncu_traffic(kernel, log2n):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{kernel}@2^{log2n}")
    except Exception:
        return None


if __name__ == "__main__":
    main()
