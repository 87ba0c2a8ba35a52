// scan.cu — parallel prefix sum (§3.2.6: "GPU-based
// parallel prefix sums (also known as `parallel scan')"), reduction
// expression "+" over int32 / int64 (wrapping, R4/R14).
//
// Single pass with decoupled look-back (BASELINE.json north_star): 8 B/elt
// for int32 (read in, write out) at the HBM roofline, instead of the
// reduce-then-scan-then-add passes of a classic three-kernel scan.
//
// Per CTA (one tile of SCAN_BLOCK x ITEMS elements, 16 KiB):
//   1. thread 0 reads the workspace epoch (acquire), then draws a tile id
//      from an atomic counter — ids are handed out in CTA start order, so
//      every predecessor tile is already running (forward progress);
//   2. each thread loads ITEMS consecutive elements with two 256-bit loads,
//      scans them serially, the block scans the thread totals (warp shuffles
//      + one shared-memory step);
//   3. the tile publishes its AGGREGATE, warp 0 looks back over up to 32
//      predecessors at a time (spinning while one is INVALID; stopping at the
//      nearest INCLUSIVE), then publishes its INCLUSIVE prefix;
//   4. the tile adds its exclusive prefix and stores with 256-bit stores.
// Look-back status words carry the call's epoch tag, so stale words of an
// earlier call read as INVALID and the workspace needs no memset per call;
// the CTA that draws the last tile id resets the counter and bumps the epoch.
// Tile 0's exclusive prefix is the carry-in c = sum(carry[0..carry_count)),
// which is how a sharded scan injects the totals of earlier shards.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ga_device.cuh"
#include "ga_host.h"

namespace ga {
namespace {

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_WARPS = SCAN_BLOCK / 32;
constexpr size_t SCAN_HEADER = 256;  // [0]: tile counter, [128]: epoch
constexpr uint32_t FLAG_INVALID = 0, FLAG_AGGREGATE = 1, FLAG_INCLUSIVE = 2;
constexpr uint32_t EPOCH_MASK = (1u << 30) - 1;

template <typename T>
constexpr int scan_items() {
  return 64 / (int)sizeof(T);  // 64 bytes per thread: two 256-bit vectors
}
template <typename T>
constexpr int64_t scan_tile() {
  return (int64_t)SCAN_BLOCK * scan_items<T>();
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Look-back status of one tile.
//  4-byte T: one 64-bit word  (epoch:30 | flag:2) << 32 | value:32 — flag and
//            value are written and read together (single-copy atomic).
//  8-byte T: a 32-bit flag word (epoch:30 | flag:2) released after the value
//            is stored in agg[] or incl[]; readers acquire the flag first.
template <typename T, int SZ = sizeof(T)>
struct Status;

template <typename T>
struct Status<T, 4> {
  uint64_t *word;
  __device__ void publish(int64_t tile, uint32_t epoch, uint32_t flag, T v) const {
    st_relaxed_u64(word + tile, ((uint64_t)((epoch << 2) | flag) << 32) | (uint32_t)v);
  }
  __device__ uint32_t read(int64_t tile, uint32_t epoch, T &v) const {
    const uint64_t w = ld_relaxed_u64(word + tile);
    const uint32_t hi = (uint32_t)(w >> 32);
    v = (T)(uint32_t)w;
    return (hi >> 2) == epoch ? (hi & 3u) : FLAG_INVALID;
  }
};

template <typename T>
struct Status<T, 8> {
  uint32_t *flag;
  T *agg;
  T *incl;
  __device__ void publish(int64_t tile, uint32_t epoch, uint32_t f, T v) const {
    (f == FLAG_INCLUSIVE ? incl : agg)[tile] = v;
    st_release_u32(flag + tile, (epoch << 2) | f);
  }
  __device__ uint32_t read(int64_t tile, uint32_t epoch, T &v) const {
    const uint32_t w = ld_acquire_u32(flag + tile);
    const uint32_t f = (w >> 2) == epoch ? (w & 3u) : FLAG_INVALID;
    if (f == FLAG_AGGREGATE) v = __ldcg(agg + tile);
    else if (f == FLAG_INCLUSIVE) v = __ldcg(incl + tile);
    return f;
  }
};

template <typename T>
struct ScanArgs {
  int64_t n;
  int64_t num_tiles;
  const T *in;
  T *out;
  const T *carry;
  int64_t carry_count;
  uint32_t *tile_counter;
  uint32_t *epoch;
  Status<T> status;
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = e_add(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Warp 0: exclusive prefix of `tile` from its predecessors' status words.
// A predecessor that stays INVALID for 10 s means a corrupted workspace (e.g.
// one shared with another kernel family): trap instead of hanging the GPU.
template <typename T>
__device__ T look_back(const Status<T> &st, int64_t tile, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  T prefix = T(0);
  int64_t pred = tile - 1;
  while (true) {
    const int64_t idx = pred - lane;  // lane 0 = nearest predecessor
    T v = T(0);
    uint32_t f = FLAG_INCLUSIVE;      // before tile 0: the neutral element
    if (idx >= 0) {
      uint32_t spins = 0;
      uint64_t t0 = 0;
      while ((f = st.read(idx, epoch, v)) == FLAG_INVALID) {
        if ((++spins & 1023u) == 0) {
          const uint64_t now = globaltimer_ns();
          if (t0 == 0) t0 = now;
          else if (now - t0 > 10000000000ull) __trap();
        }
      }
    }
    const uint32_t incl_mask = __ballot_sync(0xffffffffu, f == FLAG_INCLUSIVE);
    if (incl_mask) {
      const int first = __ffs(incl_mask) - 1;  // nearest INCLUSIVE predecessor
      prefix = e_add(prefix, warp_sum<T>(lane <= first ? v : T(0)));
      return prefix;
    }
    prefix = e_add(prefix, warp_sum<T>(v));
    pred -= 32;
  }
}

template <typename T, bool EXCLUSIVE, bool VECTOR, bool NC>
__global__ void __launch_bounds__(SCAN_BLOCK) scan_kernel(ScanArgs<T> p) {
  constexpr int ITEMS = scan_items<T>();
  constexpr int64_t TILE = scan_tile<T>();
  constexpr int NV = ITEMS * (int)sizeof(T) / 32;  // 256-bit vectors per thread
  constexpr int PER_V = 32 / (int)sizeof(T);
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ T s_warp[SCAN_WARPS];
  __shared__ T s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    const uint32_t e = ld_acquire_u32(p.epoch) & EPOCH_MASK;  // before drawing the tile id
    const uint32_t t = atomicAdd(p.tile_counter, 1u);
    if ((int64_t)t == p.num_tiles - 1) {
      // Every CTA has read the epoch and drawn its id: reset for the next call.
      *p.tile_counter = 0u;
      *p.epoch = (e + 1u) & EPOCH_MASK;
    }
    s_tile = t;
    s_epoch = e;
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const uint32_t epoch = s_epoch;
  const int64_t i0 = tile * TILE + (int64_t)threadIdx.x * ITEMS;
  const bool full = tile * TILE + TILE <= p.n;

  // 1. load ITEMS consecutive elements (out of range -> neutral 0)
  T x[ITEMS];
  if (VECTOR && full) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const V32 v = ld_vec<NC>(p.in + i0 + j * PER_V);
#pragma unroll
      for (int k = 0; k < PER_V; ++k) x[j * PER_V + k] = vget<T>(v, k);
    }
  } else {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) x[k] = (i0 + k < p.n) ? p.in[i0 + k] : T(0);
  }

  // 2. thread-serial inclusive scan, then block-wide exclusive scan of totals
#pragma unroll
  for (int k = 1; k < ITEMS; ++k) x[k] = e_add(x[k], x[k - 1]);
  const T total = x[ITEMS - 1];
  T incl = total;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl = e_add(incl, u);
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = lane < SCAN_WARPS ? s_warp[lane] : T(0);
#pragma unroll
    for (int off = 1; off < SCAN_WARPS; off <<= 1) {
      const T u = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w = e_add(w, u);
    }
    const T block_total = __shfl_sync(0xffffffffu, w, SCAN_WARPS - 1);
    if (lane < SCAN_WARPS) s_warp[lane] = w;  // inclusive over warps

    // 3. decoupled look-back
    T prefix;
    if (tile == 0) {
      prefix = T(0);
      if (lane == 0)
        for (int64_t c = 0; c < p.carry_count; ++c) prefix = e_add(prefix, p.carry[c]);
      prefix = __shfl_sync(0xffffffffu, prefix, 0);
      if (lane == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, e_add(prefix, block_total));
    } else {
      if (lane == 0) p.status.publish(tile, epoch, FLAG_AGGREGATE, block_total);
      prefix = look_back<T>(p.status, tile, epoch);
      if (lane == 0) p.status.publish(tile, epoch, FLAG_INCLUSIVE, e_add(prefix, block_total));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  const T warp_excl = warp > 0 ? s_warp[warp - 1] : T(0);
  // exclusive prefix of this thread's first element
  const T base = e_add(e_add(s_prefix, warp_excl), e_sub(incl, total));

  // 4. add the prefix and store
  T y[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if constexpr (EXCLUSIVE) y[k] = k == 0 ? base : e_add(base, x[k - 1]);
    else y[k] = e_add(base, x[k]);
  }
  if (VECTOR && full) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      V32 v;
#pragma unroll
      for (int k = 0; k < PER_V; ++k) vset<T>(v, k, y[j * PER_V + k]);
      st_256(p.out + i0 + j * PER_V, v);
    }
  } else {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k)
      if (i0 + k < p.n) p.out[i0 + k] = y[k];
  }
}

template <typename T>
size_t ws_bytes(int64_t n) {
  const int64_t tiles = cdiv(n, scan_tile<T>());
  if (sizeof(T) == 4) return SCAN_HEADER + (size_t)tiles * 8;
  return SCAN_HEADER + (size_t)cdiv(tiles * 4, 16) * 16 + (size_t)tiles * 16;
}

template <typename T, bool EXCLUSIVE>
ga_status_t run(int64_t n, const void *in, void *out, const void *carry, int64_t carry_count, void *ws,
                cudaStream_t s) {
  ScanArgs<T> p;
  p.n = n;
  p.num_tiles = cdiv(n, scan_tile<T>());
  p.in = static_cast<const T *>(in);
  p.out = static_cast<T *>(out);
  p.carry = static_cast<const T *>(carry);
  p.carry_count = carry_count;
  char *w = static_cast<char *>(ws);
  p.tile_counter = reinterpret_cast<uint32_t *>(w);
  p.epoch = reinterpret_cast<uint32_t *>(w + 128);
  if constexpr (sizeof(T) == 4) {
    p.status.word = reinterpret_cast<uint64_t *>(w + SCAN_HEADER);
  } else {
    p.status.flag = reinterpret_cast<uint32_t *>(w + SCAN_HEADER);
    char *vals = w + SCAN_HEADER + cdiv(p.num_tiles * 4, 16) * 16;
    p.status.agg = reinterpret_cast<T *>(vals);
    p.status.incl = reinterpret_cast<T *>(vals + p.num_tiles * 8);
  }
  if (p.num_tiles > 0x7fffffffLL) return fail(GA_ERR_UNSUPPORTED, "scan: n too large (%lld)", (long long)n);
  const bool vector = ((uintptr_t)in & 31) == 0 && ((uintptr_t)out & 31) == 0;
  const bool inplace = in == out;
  const int grid = (int)p.num_tiles;
  if (vector && !inplace) scan_kernel<T, EXCLUSIVE, true, true><<<grid, SCAN_BLOCK, 0, s>>>(p);
  else if (vector) scan_kernel<T, EXCLUSIVE, true, false><<<grid, SCAN_BLOCK, 0, s>>>(p);
  else scan_kernel<T, EXCLUSIVE, false, false><<<grid, SCAN_BLOCK, 0, s>>>(p);
  count_launch();
  return check_launch("scan_kernel");
}

}  // namespace

size_t scan_workspace_bytes(ga_dtype_t dt, int64_t n) {
  switch (dt) {
    case GA_I32: return ws_bytes<int32_t>(n);
    case GA_I64: return ws_bytes<int64_t>(n);
    default: return 0;
  }
}

ga_status_t launch_scan(ga_scan_kind_t kind, ga_dtype_t dt, int64_t n, const void *in, void *out,
                        const void *carry, int64_t carry_count, void *ws, cudaStream_t s) {
  const bool ex = kind == GA_SCAN_EXCLUSIVE;
  switch (dt) {
    case GA_I32:
      return ex ? run<int32_t, true>(n, in, out, carry, carry_count, ws, s)
                : run<int32_t, false>(n, in, out, carry, carry_count, ws, s);
    case GA_I64:
      return ex ? run<int64_t, true>(n, in, out, carry, carry_count, ws, s)
                : run<int64_t, false>(n, in, out, carry, carry_count, ws, s);
    default: return fail(GA_ERR_UNSUPPORTED, "scan dtype %d not instantiated", (int)dt);
  }
}

}  // namespace ga
