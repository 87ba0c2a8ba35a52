// scan_l2p.cuh — tuning lab only: persistent look-ahead variant of the
// two-touch scan (measured slower than scan_l2_kernel: 4.9 vs 5.2-5.3 TB/s
// at n = 2^28 int32, the doubled L2 footprint costs more re-read misses than
// the shorter look-back saves).  Uses the product's scan machinery.
#pragma once
#include "scan_kernel.cuh"

namespace ga {
namespace scan_detail {

// ===========================================================================
// Persistent look-ahead variant of the two-touch kernel: CTAs stay resident
// and process super-tiles in claim order with a one-tile look-ahead —
//   phase 1 of the NEXT super-tile (fold + publish its AGGREGATE) runs before
//   the look-back of the CURRENT one, so by the time warp 0 looks back the
//   predecessors have long published and the wait is about one round trip;
//   then phase 3 of the current super-tile (L2 re-read, scan, store).
// Each CTA makes exactly one failing claim; the globally last claim
// (num_tiles + grid - 1) resets the ticket.
// ===========================================================================
template <int OP, typename T, int WARPS, int ROWS, int UNROLL, int DEPTH, bool NC, bool EXCLUSIVE>
__global__ void __launch_bounds__(WARPS * 32) scan_l2p_kernel(ScanArgs<T> p) {
  using O = Op<OP, T>;
  constexpr int E = Chunk<T>::E;
  constexpr int ROW = 32 * E;
  constexpr int64_t TILE = (int64_t)WARPS * ROWS * ROW;
  static_assert(ROWS % UNROLL == 0, "ROWS must be a multiple of UNROLL");
  static_assert(WARPS <= 32, "slice folds are scanned by one warp");
  __shared__ long long s_claim[2];
  __shared__ uint32_t s_epoch;
  __shared__ T s_slice[2][WARPS];  // [buf]: slice folds, then slice exclusive prefixes
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T neutral = O::neutral();
  const int64_t last_claim = p.num_tiles + (int64_t)gridDim.x - 1;
  const uint64_t keep = l2::policy_evict_last();
  const uint64_t drop = l2::policy_evict_first();

  auto claim = [&](int buf) {  // thread 0
    const unsigned long long old = atomicAdd(p.ticket, 1ull);
    const int64_t t = (int64_t)(uint32_t)old;
    const uint32_t e = (uint32_t)(old >> 32) & EPOCH_MASK;
    if (t == last_claim) *p.ticket = (unsigned long long)((e + 1u) & EPOCH_MASK) << 32;
    s_epoch = e;
    s_claim[buf] = t < p.num_tiles ? (long long)t : -1ll;
  };
  auto load_row = [&](int64_t tile, int r, uint64_t pol, T (&v)[E]) {
    const int64_t i = tile * TILE + (int64_t)warp * ROWS * ROW + (int64_t)r * ROW + lane * E;
    if ((tile + 1) * TILE <= p.n) {
      Chunk<T>::unpack(l2::ldg128_hint<NC>(p.in + i, pol), v);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = i + k < p.n ? p.in[i + k] : neutral;
    }
  };
  // phase 1 of `tile` into s_slice[buf]; warp 0 then publishes the aggregate
  auto phase1 = [&](int64_t tile, int buf, uint32_t epoch) {
    T acc = neutral;
#pragma unroll 1
    for (int r0 = 0; r0 < ROWS; r0 += UNROLL) {
      T v[UNROLL][E];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) load_row(tile, r0 + u, keep, v[u]);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
#pragma unroll
        for (int k = 0; k < E; ++k) acc = O::fold(acc, v[u][k]);
    }
    acc = warp_fold<OP, T>(acc);
    if (lane == 0) s_slice[buf][warp] = acc;
    __syncthreads();
    if (warp == 0) {
      const T mine = lane < WARPS ? s_slice[buf][lane] : neutral;
      const T w = warp_inclusive<OP, T>(mine, lane);
      const T total = __shfl_sync(0xffffffffu, w, WARPS - 1);
      if (lane == 0) {
        if (tile == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, O::fold(carry_in<OP, T>(p), total));
        else p.status.publish(tile, epoch, FLAG_AGGREGATE, total);
      }
    }
  };
  // look-back for `tile` (warp 0) -> s_slice[buf] = slice exclusive prefixes
  auto lookback = [&](int64_t tile, int buf, uint32_t epoch) {
    if (warp == 0) {
      const T mine = lane < WARPS ? s_slice[buf][lane] : neutral;
      const T w = warp_inclusive<OP, T>(mine, lane);
      const T wex = warp_exclusive_of<OP, T>(w, lane);
      const T total = __shfl_sync(0xffffffffu, w, WARPS - 1);
      T prefix;
      if (tile == 0) {
        prefix = lane == 0 ? carry_in<OP, T>(p) : neutral;
        prefix = __shfl_sync(0xffffffffu, prefix, 0);
      } else {
        prefix = look_back<OP, T, DEPTH>(p.status, tile, epoch);
        if (lane == 0) p.status.publish(tile, epoch, FLAG_INCLUSIVE, O::fold(prefix, total));
      }
      __syncwarp();
      if (lane < WARPS) s_slice[buf][lane] = O::fold(prefix, wex);
    }
  };
  auto phase3 = [&](int64_t tile, int buf) {
    const int64_t slice0 = tile * TILE + (int64_t)warp * ROWS * ROW;
    const bool full = (tile + 1) * TILE <= p.n;
    T base = s_slice[buf][warp];
#pragma unroll 1
    for (int r0 = 0; r0 < ROWS; r0 += UNROLL) {
      T v[UNROLL][E];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) load_row(tile, r0 + u, drop, v[u]);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
#pragma unroll
        for (int k = 1; k < E; ++k) v[u][k] = O::fold(v[u][k - 1], v[u][k]);
        const T x = warp_inclusive<OP, T>(v[u][E - 1], lane);
        const T cb = O::fold(base, warp_exclusive_of<OP, T>(x, lane));
        base = O::fold(base, __shfl_sync(0xffffffffu, x, 31));
        T o[E];
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if constexpr (EXCLUSIVE) o[k] = k == 0 ? cb : O::fold(cb, v[u][k - 1]);
          else o[k] = O::fold(cb, v[u][k]);
        }
        const int64_t i = slice0 + (int64_t)(r0 + u) * ROW + lane * E;
        if (full) {
          l2::stg128_hint(p.out + i, Chunk<T>::pack(o), drop);
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k)
            if (i + k < p.n) p.out[i + k] = o[k];
        }
      }
    }
  };

  if (threadIdx.x == 0) claim(0);
  __syncthreads();
  int cur = 0;
  int64_t t_cur = s_claim[0];
  uint32_t epoch = s_epoch;
  if (t_cur < 0) return;
  phase1(t_cur, cur, epoch);
  while (true) {
    // claim and fold the next super-tile before looking back for this one
    __syncthreads();  // s_claim[cur^1] / s_slice[cur^1] free (used two iterations ago)
    if (threadIdx.x == 0) claim(cur ^ 1);
    __syncthreads();
    const int64_t t_next = s_claim[cur ^ 1];
    if (t_next >= 0) phase1(t_next, cur ^ 1, epoch);
    lookback(t_cur, cur, epoch);
    __syncthreads();
    phase3(t_cur, cur);
    if (t_next < 0) return;
    t_cur = t_next;
    cur ^= 1;
  }
}

}  // namespace scan_detail
}  // namespace ga
