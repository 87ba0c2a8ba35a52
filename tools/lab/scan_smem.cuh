// scan_smem.cuh — the single-touch scan kernel (round 2): each CTA brings
// its tile into shared memory with the TMA unit (cp.async.bulk, one
// mbarrier per warp slice), so every element crosses HBM exactly once in
// each direction and the L2 only passes data through (the two-touch
// scan_l2_kernel re-reads each tile from L2, which costs L2 capacity and
// re-read misses at large tiles; profiles/r2_scan.md).  Several CTAs share
// an SM, so while one waits for its look-back the others stream.
//
//   load     lane 0 of data warp w issues one bulk copy of slice w
//            (global -> shared, L2 evict_first) on mbarrier w; the ragged
//            last tile is loaded with guarded scalar loads instead;
//   phase 1  warp w folds its slice (from shared memory); slice totals go to
//            the look-back warp;
//   phase 2  the look-back warp (one extra warp) turns them into the tile
//            AGGREGATE, publishes it, looks back (scan_kernel.cuh) and
//            publishes INCLUSIVE; meanwhile every data warp scans its slice
//            in place (local prefix, relative to the slice start) and, with
//            PF, asks the TMA unit to prefetch its slice of the tile pf_dist
//            ids ahead into L2;
//   phase 3  out = prefix(slice) (+) local prefix, read from shared memory,
//            stored 512 bytes per warp instruction (STG.128, evict_first).
// Results: the same fold order as scan_l2_kernel within rows (in-lane serial,
// warp shuffle, rows serial), so integer and max/min scans are exact and
// float SUM stays within DESIGN.md R22's bound.
#pragma once
#include "scan_kernel.cuh"  // product machinery (csrc/)

namespace ga {
namespace scan_detail {

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// Bulk copy global -> shared of `bytes` (multiple of 16, 16-byte aligned on
// both sides), completion counted on `bar` (armed here with the byte count).
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// DW data warps (+1 look-back warp), SLICE input bytes per data warp (a
// multiple of 512: SLICE/512 rows of 32 lanes x 16 bytes).
template <int OP, typename T, int DW, int SLICE, int DEPTH, bool NC, bool EXCLUSIVE, bool PF, bool TRACE = false,
          bool STMA = false, bool SRV = false>
__global__ void __launch_bounds__((DW + 1) * 32) scan_smem_kernel(ScanArgs<T, T> p, uint64_t *trace = nullptr) {
  using O = Op<OP, T>;
  constexpr int E = Chunk<T>::E;        // elements per lane per row
  constexpr int ROW = 32 * E;           // elements per 512-byte row
  constexpr int ROWS = SLICE / 512;     // rows per slice
  constexpr int64_t TILE = (int64_t)DW * ROWS * ROW;
  static_assert(SLICE % 512 == 0 && DW <= 32, "slice shape");
  extern __shared__ __align__(128) uint4 s_data[];  // DW * SLICE bytes
  __shared__ __align__(8) uint64_t s_bar[DW];
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ T s_slice[DW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T neutral = O::neutral();

  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int w = 0; w < DW; ++w) mbar_init(&s_bar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t t, e;
    draw_tile(p, t, e);
    s_tile = t;
    s_epoch = e;
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const uint32_t epoch = s_epoch;
  const bool full = tile * TILE + TILE <= p.n;
  const int64_t slice0 = tile * TILE + (int64_t)warp * ROWS * ROW;  // first element of my slice
  uint4 *mine = s_data + (size_t)warp * (SLICE / 16) + lane;         // my 16 bytes of row 0
  auto stamp = [&](int k) {
    if constexpr (TRACE) trace[tile * 8 + k] = globaltimer_ns();
  };
  if (TRACE && threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    trace[tile * 8 + 7] = sm;
    stamp(0);
  }

  if (warp < DW) {
    if (full) {
      if (lane == 0) bulk_load(s_data + (size_t)warp * (SLICE / 16), p.in + slice0, SLICE, &s_bar[warp],
                               l2::policy_evict_first());
      mbar_wait(&s_bar[warp], 0);
      if (TRACE && lane == 0 && warp == DW - 1) stamp(1);
    } else {
#pragma unroll 1
      for (int r = 0; r < ROWS; ++r) {
        T e[E];
        const int64_t i = slice0 + (int64_t)r * ROW + lane * E;
#pragma unroll
        for (int k = 0; k < E; ++k) e[k] = i + k < p.n ? p.in[i + k] : neutral;
        mine[r * 32] = Chunk<T>::pack(e);
      }
      __syncwarp();
    }
    // phase 1: slice fold
    T acc = neutral;
#pragma unroll 4
    for (int r = 0; r < ROWS; ++r) {
      T v[E];
      Chunk<T>::unpack(mine[r * 32], v);
#pragma unroll
      for (int k = 0; k < E; ++k) acc = O::fold(acc, v[k]);
    }
    acc = warp_fold<OP, T>(acc);
    if (lane == 0) s_slice[warp] = acc;
  }
  __syncthreads();

  if (warp == DW) {
    // phase 2, look-back warp: slice prefixes, aggregate, look-back
    const T m = lane < DW ? s_slice[lane] : neutral;
    const T w = warp_inclusive<OP, T>(m, lane);
    const T wex = warp_exclusive_of<OP, T>(w, lane);
    const T total = __shfl_sync(0xffffffffu, w, DW - 1);
    T prefix;
    if (tile == 0) {
      prefix = lane == 0 ? carry_in<OP, T>(p) : neutral;
      prefix = __shfl_sync(0xffffffffu, prefix, 0);
      if (lane == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, O::fold(prefix, total));
    } else if constexpr (SRV) {
      // prefix server (tile 0's CTA, below) publishes every tile's INCLUSIVE
      // in order: publish the AGGREGATE, then wait for the predecessor's
      // INCLUSIVE — one status word, polled by lane 0
      if (lane == 0) p.status.publish(tile, epoch, FLAG_AGGREGATE, total);
      if (TRACE && lane == 0) stamp(2);
      T pv = neutral;
      if (lane == 0) {
        uint32_t f, spins = 0;
        uint64_t t0 = 0;
        while ((f = p.status.read(tile - 1, epoch, pv)) != FLAG_INCLUSIVE) {
          if ((++spins & 1023u) == 0) {
            const uint64_t now = globaltimer_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 5000000000ull) __trap();  // lab guard: never hang the box
          }
        }
      }
      prefix = __shfl_sync(0xffffffffu, pv, 0);
      if (TRACE && lane == 0) stamp(3);
    } else {
      if (lane == 0) p.status.publish(tile, epoch, FLAG_AGGREGATE, total);
      if (TRACE && lane == 0) stamp(2);
      prefix = look_back<OP, T, DEPTH>(p.status, tile, epoch);
      if (lane == 0) p.status.publish(tile, epoch, FLAG_INCLUSIVE, O::fold(prefix, total));
      if (TRACE && lane == 0) stamp(3);
    }
    if (lane < DW) s_slice[lane] = O::fold(prefix, wex);  // exclusive prefix of slice `lane`
  } else {
    if constexpr (PF) {
      const int64_t nt = tile + p.pf_dist;
      if (lane == 0 && (nt + 1) * TILE <= p.n)
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(
                         p.in + nt * TILE + (int64_t)warp * ROWS * ROW),
                     "r"((uint32_t)SLICE), "l"(l2::policy_evict_last())
                     : "memory");
    }
    // phase 2, data warps: local scan of the slice, in place
    T run = neutral;
#pragma unroll 2
    for (int r = 0; r < ROWS; ++r) {
      T v[E], o[E];
      Chunk<T>::unpack(mine[r * 32], v);
#pragma unroll
      for (int k = 1; k < E; ++k) v[k] = O::fold(v[k - 1], v[k]);
      const T x = warp_inclusive<OP, T>(v[E - 1], lane);
      const T cb = O::fold(run, warp_exclusive_of<OP, T>(x, lane));
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if constexpr (EXCLUSIVE) o[k] = k == 0 ? cb : O::fold(cb, v[k - 1]);
        else o[k] = O::fold(cb, v[k]);
      }
      mine[r * 32] = Chunk<T>::pack(o);
      run = O::fold(run, __shfl_sync(0xffffffffu, x, 31));
    }
  }
  __syncthreads();
  if (warp == DW) {
    if constexpr (SRV) {
      if (tile == 0) {
        // The prefix server: a sliding window of 32 tiles; every poll takes
        // the run of consecutive published AGGREGATEs from the window start,
        // scans it onto the running prefix and publishes their INCLUSIVEs.
        T run = neutral;
        if (lane == 0) {
          T v0;
          p.status.read(0, epoch, v0);
          run = v0;
        }
        run = __shfl_sync(0xffffffffu, run, 0);
        int64_t next = 1;
        const int64_t last = p.num_tiles - 1;  // nobody needs the last tile's INCLUSIVE
        uint64_t t0 = globaltimer_ns();
        while (next < last) {
          if (globaltimer_ns() - t0 > 5000000000ull) __trap();  // lab guard: never hang the box
          const int64_t t = next + lane;
          T v = neutral;
          uint32_t f = FLAG_INVALID;
          if (t < last) f = p.status.read(t, epoch, v);
          const uint32_t ready = __ballot_sync(0xffffffffu, t < last && f != FLAG_INVALID);
          const int cnt = __ffs(~ready) - 1 < 0 ? 32 : __ffs(~ready) - 1;  // leading ready lanes
          if (cnt == 0) continue;
          const T x = warp_inclusive<OP, T>(lane < cnt ? v : neutral, lane);
          if (lane < cnt) p.status.publish(t, epoch, FLAG_INCLUSIVE, O::fold(run, x));
          run = O::fold(run, __shfl_sync(0xffffffffu, x, cnt - 1));
          next += cnt;
        }
      }
    }
    return;
  }

  // phase 3: add the slice prefix and store
  const T base = s_slice[warp];
  const uint64_t drop = l2::policy_evict_first();
  if (STMA && full) {
    // final values back into shared memory, then one bulk store per slice
#pragma unroll 4
    for (int r = 0; r < ROWS; ++r) {
      T o[E];
      Chunk<T>::unpack(mine[r * 32], o);
#pragma unroll
      for (int k = 0; k < E; ++k) o[k] = O::fold(base, o[k]);
      mine[r * 32] = Chunk<T>::pack(o);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                       p.out + slice0),
                   "r"(smem_u32(s_data + (size_t)warp * (SLICE / 16))), "r"((uint32_t)SLICE), "l"(drop)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    if (TRACE && warp == 0 && lane == 0) stamp(4);
    return;
  }
#pragma unroll 4
  for (int r = 0; r < ROWS; ++r) {
    T o[E];
    Chunk<T>::unpack(mine[r * 32], o);
#pragma unroll
    for (int k = 0; k < E; ++k) o[k] = O::fold(base, o[k]);
    const int64_t i = slice0 + (int64_t)r * ROW + lane * E;
    if (full) {
      l2::stg128_hint(p.out + i, Chunk<T>::pack(o), drop);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (i + k < p.n) p.out[i + k] = o[k];
    }
  }
  if (TRACE && warp == 0 && lane == 0) stamp(4);
  (void)NC;
}

}  // namespace scan_detail
}  // namespace ga
