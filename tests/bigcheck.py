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
