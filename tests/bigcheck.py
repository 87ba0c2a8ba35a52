"""Chunked, multi-process oracle evaluation for the full-size (BASELINE.json
configs) parity tests.  TEST INFRASTRUCTURE: imports only numpy, synth and
the oracle (no torch), so spawn-started workers are cheap.

Every chunk regenerates its inputs from the counter-based generator (no
host array of the full n is ever built) and calls the plain oracle on it;
the per-chunk results are then combined:
  float SUM  -> math.fsum of the per-chunk (near-exact, Neumaier) partials
  int SUM    -> Python big-int sum, wrapped to the output width
  MAX / MIN  -> max / min of the chunk extremes."""
import math
import multiprocessing as mp
import os

import numpy as np

CHUNK = 1 << 25


def _job(args):
    import oracle
    import synth
    (kind, seed, lo, hi, kind_y, seed_y, start, m, op, map_, out_dtype) = args
    x = synth.host_fill(kind, seed, m, start=start, lo=lo, hi=hi)
    y = synth.host_fill(kind_y, seed_y, m, start=start) if kind_y is not None else None
    odt = np.dtype(out_dtype) if out_dtype else None
    if op == oracle.SUM and x.dtype.kind == "f":
        v, sa = oracle.reduce(op, map_, x, y, return_sumabs=True)
        return float(v), float(sa)
    return oracle.reduce(op, map_, x, y, out_dtype=odt), None


def chunked_reduce(op, map_, n, kind, seed, lo=0, hi=0, kind_y=None, seed_y=0, out_dtype=None, procs=None):
    """Oracle reduction of generator stream(s) over [0, n).  Returns
    (value, sum|t_i| or None)."""
    import oracle
    jobs = [(kind, seed, lo, hi, kind_y, seed_y, s, min(CHUNK, n - s), op, map_, out_dtype)
            for s in range(0, n, CHUNK)]
    procs = procs or max(1, min(len(os.sched_getaffinity(0)), 32))
    with mp.get_context("spawn").Pool(procs) as pool:
        parts = pool.map(_job, jobs, chunksize=1)
    vals = [p[0] for p in parts]
    if op == oracle.SUM:
        if isinstance(vals[0], float):
            return math.fsum(vals), math.fsum(p[1] for p in parts)
        w = np.dtype(out_dtype).itemsize * 8 if out_dtype else 64
        v = sum(vals) % (1 << w)
        return (v - (1 << w) if v >= 1 << (w - 1) else v), None
    return (max(vals) if op == oracle.MAX else min(vals)), None


def chunk_sums_int(n, kind, seed, lo, hi, chunk, procs=None):
    """Exact integer sums of every `chunk`-sized block of the stream (Python ints)."""
    import oracle
    jobs = [(kind, seed, lo, hi, None, 0, s, min(chunk, n - s), oracle.SUM, oracle.MAP_ID, "int64")
            for s in range(0, n, chunk)]
    procs = procs or max(1, min(len(os.sched_getaffinity(0)), 32))
    with mp.get_context("spawn").Pool(procs) as pool:
        parts = pool.map(_job, jobs, chunksize=1)
    return [int(p[0]) for p in parts]


def _scan_cmp_job(args):
    """Compare one chunk of a GPU scan output (already in shared memory)
    element by element with the oracle's scan of the regenerated chunk."""
    from multiprocessing import shared_memory
    import oracle
    import synth
    (shm_name, off, kind, seed, lo, hi, start, m, carry, exclusive, out_dtype) = args
    odt = np.dtype(out_dtype)
    shm = shared_memory.SharedMemory(name=shm_name)
    try:
        got = np.ndarray((m,), dtype=odt, buffer=shm.buf, offset=off)
        x = synth.host_fill(kind, seed, m, start=start, lo=lo, hi=hi)
        ref = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x, carry=odt.type(carry),
                          out_dtype=odt if odt != x.dtype else None)
        bad = np.flatnonzero(got != ref)
        res = (start, int(bad.size), int(start + bad[0]) if bad.size else -1)
        del got
        return res
    finally:
        shm.close()


def chunked_scan_compare(fetch, n, kind, seed, lo, hi, out_dtype, exclusive, chunk=CHUNK, batch=32, procs=None):
    """Element-by-element comparison of a whole integer scan output of n
    elements against the chunked oracle: every chunk's carry-in is the exact
    (wrapped) sum of the chunks before it, and the oracle scans each
    regenerated chunk from that carry.  `fetch(start, m, dest)` copies output
    elements [start, start+m) into the numpy array `dest`.  The output
    streams through a shared-memory window of `batch` chunks.  Returns
    (elements compared, mismatches, first mismatching index or -1)."""
    from multiprocessing import shared_memory
    odt = np.dtype(out_dtype)
    w = 1 << (odt.itemsize * 8)
    sums = chunk_sums_int(n, kind, seed, lo, hi, chunk, procs=procs)
    carries, prefix = [], 0
    for s in sums:
        carries.append(((prefix + w // 2) % w) - w // 2)
        prefix += s
    starts = list(range(0, n, chunk))
    procs = procs or max(1, min(len(os.sched_getaffinity(0)), 32))
    shm = shared_memory.SharedMemory(create=True, size=batch * chunk * odt.itemsize)
    compared, mismatches, first = 0, 0, -1
    try:
        with mp.get_context("spawn").Pool(procs) as pool:
            for b0 in range(0, len(starts), batch):
                jobs = []
                for j, start in enumerate(starts[b0:b0 + batch]):
                    m = min(chunk, n - start)
                    off = j * chunk * odt.itemsize
                    fetch(start, m, np.ndarray((m,), dtype=odt, buffer=shm.buf, offset=off))
                    jobs.append((shm.name, off, kind, seed, lo, hi, start, m, carries[b0 + j], exclusive, odt.str))
                for start, bad, idx in pool.map(_scan_cmp_job, jobs, chunksize=1):
                    compared += min(chunk, n - start)
                    mismatches += bad
                    if bad and (first < 0 or idx < first):
                        first = idx
    finally:
        shm.close()
        shm.unlink()
    return compared, mismatches, first


def _chunk_sum_abs_job(args):
    import oracle
    import synth
    kind, seed, start, m = args
    x = synth.host_fill(kind, seed, m, start=start)
    v, sa = oracle.reduce(oracle.SUM, oracle.MAP_ID, x, return_sumabs=True)
    return float(v), float(sa)


def _float_scan_cmp_job(args):
    """One chunk of a float SUM scan against the oracle's exact prefix sums
    within DESIGN.md R22's bound, global index i: |gpu_i - S_i| <=
    (i/2048 + 512) * u * (sum_{j<=i} |x_j|)."""
    from multiprocessing import shared_memory
    import oracle
    import synth
    (shm_name, off, kind, seed, start, m, carry, abs_carry, exclusive, out_dtype, u) = args
    odt = np.dtype(out_dtype)
    shm = shared_memory.SharedMemory(name=shm_name)
    try:
        got = np.ndarray((m,), dtype=odt, buffer=shm.buf, offset=off).astype(np.float64)
        x = synth.host_fill(kind, seed, m, start=start)
        ref, sa = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x, carry=carry,
                              return_sumabs=True)
        sa_global = abs_carry + (sa - abs(carry))
        lim = ((start + np.arange(m, dtype=np.float64)) / 2048.0 + 512.0) * u * sa_global + 1e-300
        err = np.abs(got - ref)
        bad = np.flatnonzero(err > lim)
        return (start, int(bad.size), int(start + bad[0]) if bad.size else -1, float(np.max(err / lim)))
    finally:
        shm.close()


def chunked_float_scan_compare(fetch, n, kind, seed, out_dtype, exclusive, chunk=CHUNK, batch=32, procs=None):
    """Every element of a float SUM scan of n elements against the chunked
    oracle: chunk c starts from the exact sum of the chunks before it (the
    oracle's Neumaier float64 chunk sums combined with math.fsum), and each
    element must lie within R22's bound.  Returns (compared, violations,
    first violating index or -1, max error / bound)."""
    from multiprocessing import shared_memory
    odt = np.dtype(out_dtype)
    u = 2.0 ** -24 if odt == np.float32 else 2.0 ** -53
    starts = list(range(0, n, chunk))
    procs = procs or max(1, min(len(os.sched_getaffinity(0)), 32))
    with mp.get_context("spawn").Pool(procs) as pool:
        parts = pool.map(_chunk_sum_abs_job, [(kind, seed, s, min(chunk, n - s)) for s in starts], chunksize=1)
    carries, abs_carries = [], []
    for c in range(len(starts)):
        carries.append(math.fsum(p[0] for p in parts[:c]))
        abs_carries.append(math.fsum(p[1] for p in parts[:c]))
    shm = shared_memory.SharedMemory(create=True, size=batch * chunk * odt.itemsize)
    compared, bad_total, first, worst = 0, 0, -1, 0.0
    try:
        with mp.get_context("spawn").Pool(procs) as pool:
            for b0 in range(0, len(starts), batch):
                jobs = []
                for j, start in enumerate(starts[b0:b0 + batch]):
                    m = min(chunk, n - start)
                    off = j * chunk * odt.itemsize
                    fetch(start, m, np.ndarray((m,), dtype=odt, buffer=shm.buf, offset=off))
                    jobs.append((shm.name, off, kind, seed, start, m, carries[b0 + j], abs_carries[b0 + j], exclusive,
                                 odt.str, u))
                for start, bad, idx, w in pool.map(_float_scan_cmp_job, jobs, chunksize=1):
                    compared += min(chunk, n - start)
                    bad_total += bad
                    worst = max(worst, w)
                    if bad and (first < 0 or idx < first):
                        first = idx
    finally:
        shm.close()
        shm.unlink()
    return compared, bad_total, first, worst
