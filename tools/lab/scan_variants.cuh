// scan_kernel.cuh — the single-pass decoupled look-back scan kernel,
// templated on its tile shape so scan.cu can instantiate the tuned
// configuration (and tools/lab can sweep others).  See scan.cu for the
// algorithm and its citations.
#pragma once
// FROZEN COPY for the tuning lab: the scan kernel variants measured while
// tuning (register-tiled, TMA-staged, warp-specialized, pipelined, two-touch),
// int SUM only.  The product kernels live in paper_1304_5553_b200/csrc/scan_kernel.cuh.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ga_device.cuh"

namespace ga {
namespace scan_lab_old {

constexpr uint32_t FLAG_INVALID = 0, FLAG_AGGREGATE = 1, FLAG_INCLUSIVE = 2;
constexpr uint32_t EPOCH_MASK = (1u << 30) - 1;
// Workspace header: one 64-bit ticket word {epoch:32 | tile counter:32} in its
// own 256-byte block; per-tile status follows.
constexpr size_t HEADER = 256;

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
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
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
  unsigned long long *ticket;  // {epoch:32 | counter:32}
  Status<T> status;
  unsigned long long *trace;   // tuning lab only: per-tile timestamps (nullptr in the product)
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = e_add(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// Spin until predecessor `idx` has published.  A predecessor that stays
// INVALID for 10 s means a corrupted workspace: trap instead of hanging.
template <typename T, int BACKOFF_NS>
__device__ __forceinline__ uint32_t wait_status(const Status<T> &st, int64_t idx, uint32_t epoch, T &v) {
  uint32_t f = st.read(idx, epoch, v);
  if (f != FLAG_INVALID) return f;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while ((f = st.read(idx, epoch, v)) == FLAG_INVALID) {
    if (BACKOFF_NS > 0) __nanosleep(BACKOFF_NS);
    if ((++spins & 1023u) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 10000000000ull) __trap();
    }
  }
  return f;
}

// Warp 0: exclusive prefix of `tile` from its predecessors' status words.
// Each round reads 32*DEPTH predecessors (DEPTH independent loads per lane in
// flight), waits until all are published, and stops at the nearest INCLUSIVE.
template <typename T, int DEPTH, int BACKOFF_NS>
__device__ T look_back(const Status<T> &st, int64_t tile, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  T prefix = T(0);
  int64_t pred = tile - 1;
  while (true) {
    T v[DEPTH];
    uint32_t f[DEPTH];
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      const int64_t idx = pred - lane - 32 * j;  // distance 1 + lane + 32 j
      v[j] = T(0);
      f[j] = FLAG_INCLUSIVE;                      // before tile 0: the neutral element
      if (idx >= 0) f[j] = st.read(idx, epoch, v[j]);
    }
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      const int64_t idx = pred - lane - 32 * j;
      if (f[j] == FLAG_INVALID) f[j] = wait_status<T, BACKOFF_NS>(st, idx, epoch, v[j]);
    }
    T part = T(0);
    bool done = false;
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      if (!done) {
        const uint32_t m = __ballot_sync(0xffffffffu, f[j] == FLAG_INCLUSIVE);
        if (m) {
          const int first = __ffs(m) - 1;  // nearest INCLUSIVE in this row
          part = e_add(part, lane <= first ? v[j] : T(0));
          done = true;
        } else {
          part = e_add(part, v[j]);
        }
      }
    }
    prefix = e_add(prefix, warp_sum<T>(part));
    if (done) return prefix;
    pred -= 32 * DEPTH;
  }
}

template <typename T, int BLOCK, int ITEMS, int DEPTH, int BACKOFF_NS, bool EXCLUSIVE, bool VECTOR, bool NC>
__global__ void __launch_bounds__(BLOCK) scan_kernel(ScanArgs<T> p) {
  constexpr int WARPS = BLOCK / 32;
  constexpr int64_t TILE = (int64_t)BLOCK * ITEMS;
  constexpr int PER_V = 32 / (int)sizeof(T);
  constexpr int NV = ITEMS / PER_V;  // 256-bit vectors per thread
  static_assert(ITEMS % PER_V == 0, "ITEMS must fill whole 256-bit vectors");
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ T s_warp[WARPS];
  __shared__ T s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    // One round trip gives both the tile id and the call's epoch.
    const unsigned long long old = atomicAdd(p.ticket, 1ull);
    const uint32_t t = (uint32_t)old, e = (uint32_t)(old >> 32) & EPOCH_MASK;
    if ((int64_t)t == p.num_tiles - 1) {
      // Every CTA has drawn its id (and with it the epoch): reset for the next call.
      *p.ticket = (unsigned long long)((e + 1u) & EPOCH_MASK) << 32;
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
    V32 raw[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) raw[j] = ld_vec<NC>(p.in + i0 + j * PER_V);
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int k = 0; k < PER_V; ++k) x[j * PER_V + k] = vget<T>(raw[j], k);
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
    T w = lane < WARPS ? s_warp[lane] : T(0);
#pragma unroll
    for (int off = 1; off < WARPS; off <<= 1) {
      const T u = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w = e_add(w, u);
    }
    const T block_total = __shfl_sync(0xffffffffu, w, WARPS - 1);
    if (lane < WARPS) s_warp[lane] = w;  // inclusive over warps

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
      prefix = look_back<T, DEPTH, BACKOFF_NS>(p.status, tile, epoch);
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
size_t status_bytes(int64_t tiles) {
  if (sizeof(T) == 4) return (size_t)tiles * 8;
  return (size_t)((tiles * 4 + 15) / 16) * 16 + (size_t)tiles * 16;
}

// Fill the argument block for a tile size of TILE elements.
template <typename T>
ScanArgs<T> make_args(int64_t n, int64_t tile_elems, const void *in, void *out, const void *carry,
                      int64_t carry_count, void *ws) {
  ScanArgs<T> p;
  p.n = n;
  p.num_tiles = (n + tile_elems - 1) / tile_elems;
  p.in = static_cast<const T *>(in);
  p.out = static_cast<T *>(out);
  p.carry = static_cast<const T *>(carry);
  p.carry_count = carry_count;
  p.trace = nullptr;
  char *w = static_cast<char *>(ws);
  p.ticket = reinterpret_cast<unsigned long long *>(w);
  if constexpr (sizeof(T) == 4) {
    p.status.word = reinterpret_cast<uint64_t *>(w + HEADER);
  } else {
    p.status.flag = reinterpret_cast<uint32_t *>(w + HEADER);
    char *vals = w + HEADER + ((p.num_tiles * 4 + 15) / 16) * 16;
    p.status.agg = reinterpret_cast<T *>(vals);
    p.status.incl = reinterpret_cast<T *>(vals + p.num_tiles * 8);
  }
  return p;
}

// ===========================================================================
// Persistent, TMA-fed variant.  One or two CTAs per SM stay resident and
// claim tiles from the same {epoch | counter} ticket; each CTA keeps STAGES
// tiles in flight in a shared-memory ring filled by 1-D bulk TMA copies
// (cp.async.bulk, completion on an mbarrier), so HBM reads continue while
// the CTA waits in the look-back of its oldest tile.  Tiles are processed
// warp-striped: every LDS.128 / STG.128 of a warp covers 512 contiguous bytes
// (conflict-free, fully coalesced); the scan order inside a warp is chunk
// row by chunk row (chunk = 16 bytes).
// ===========================================================================
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for the phase with the given parity to complete.  A barrier that
// never completes (a bug or a corrupted workspace) traps after 10 s instead
// of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++spins & 255u) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 10000000000ull) __trap();
    }
  }
}
// Generic-proxy accesses of shared memory before this point are ordered
// before later async-proxy (TMA) writes to it.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void bulk_load(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ uint4 lds128(const void *p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void stg128(void *p, const uint4 &v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

template <typename T>
struct Chunk;  // 16 bytes viewed as E elements
template <>
struct Chunk<int32_t> {
  static constexpr int E = 4;
  __device__ static void unpack(const uint4 &v, int32_t (&e)[4]) {
    e[0] = (int32_t)v.x;
    e[1] = (int32_t)v.y;
    e[2] = (int32_t)v.z;
    e[3] = (int32_t)v.w;
  }
  __device__ static uint4 pack(const int32_t (&e)[4]) {
    return make_uint4((uint32_t)e[0], (uint32_t)e[1], (uint32_t)e[2], (uint32_t)e[3]);
  }
};
template <>
struct Chunk<int64_t> {
  static constexpr int E = 2;
  __device__ static void unpack(const uint4 &v, int64_t (&e)[2]) {
    e[0] = (int64_t)(((uint64_t)v.y << 32) | v.x);
    e[1] = (int64_t)(((uint64_t)v.w << 32) | v.z);
  }
  __device__ static uint4 pack(const int64_t (&e)[2]) {
    return make_uint4((uint32_t)(uint64_t)e[0], (uint32_t)((uint64_t)e[0] >> 32), (uint32_t)(uint64_t)e[1],
                      (uint32_t)((uint64_t)e[1] >> 32));
  }
};

}  // namespace tma

// BLOCK threads, CH 16-byte chunks per thread per tile -> TILE_BYTES =
// BLOCK*CH*16; STAGES tiles in the ring.  Requires in/out 16-byte aligned.
template <typename T, int BLOCK, int CH, int STAGES, int DEPTH, bool EXCLUSIVE>
__global__ void __launch_bounds__(BLOCK) scan_tma_kernel(ScanArgs<T> p) {
  using namespace tma;
  constexpr int WARPS = BLOCK / 32;
  constexpr int E = Chunk<T>::E;
  constexpr int TILE_BYTES = BLOCK * CH * 16;
  constexpr int64_t TILE = TILE_BYTES / (int)sizeof(T);
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full_bar[STAGES];
  __shared__ long long stage_tile[STAGES];
  __shared__ uint32_t s_epoch;
  __shared__ int s_done;
  __shared__ T s_warp[2][WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t last_claim = p.num_tiles + (int64_t)gridDim.x - 1;

  // Producer (warp 1 lane 0, or thread 0 when BLOCK == 32): claim a tile and
  // start its bulk copy into stage s, or mark s empty when the work is done.
  auto refill = [&](int s) {
    if (!s_done) {
      const unsigned long long old = atomicAdd(p.ticket, 1ull);
      const int64_t t = (int64_t)(uint32_t)old;
      const uint32_t e = (uint32_t)(old >> 32) & EPOCH_MASK;
      s_epoch = e;
      if (t == last_claim) *p.ticket = (unsigned long long)((e + 1u) & EPOCH_MASK) << 32;
      if (t < p.num_tiles) {
        stage_tile[s] = t;
        if (p.trace) p.trace[t * 8 + 0] = globaltimer_ns();
        if ((t + 1) * TILE <= p.n) {
          fence_proxy_async();
          mbar_arrive_expect_tx(&full_bar[s], TILE_BYTES);
          bulk_load(ring + (size_t)s * TILE_BYTES, p.in + t * TILE, TILE_BYTES, &full_bar[s]);
        } else {
          mbar_arrive(&full_bar[s]);  // ragged last tile: consumers read global memory
        }
        return;
      }
      s_done = 1;  // exactly one failed claim per CTA (the reset count relies on it)
    }
    stage_tile[s] = -1;
    mbar_arrive(&full_bar[s]);
  };

  const int producer = WARPS > 1 ? 32 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full_bar[s], 1);
    s_done = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == producer)
    for (int s = 0; s < STAGES; ++s) refill(s);

  uint32_t phase = 0;
  for (int it = 0, stage = 0;; ++it) {
    mbar_wait(&full_bar[stage], phase);
    const long long tile = stage_tile[stage];
    if (tile < 0) break;
    const uint32_t epoch = s_epoch;
    const int buf = it & 1;
    const int64_t tile0 = (int64_t)tile * TILE;
    const bool full = tile0 + TILE <= p.n;

    // 1. warp-striped chunk loads: chunk (warp*CH + j)*32 + lane
    T v[CH][E];
    if (full) {
      const uint8_t *base = ring + (size_t)stage * TILE_BYTES;
#pragma unroll
      for (int j = 0; j < CH; ++j) Chunk<T>::unpack(lds128(base + ((warp * CH + j) * 32 + lane) * 16), v[j]);
    } else {
#pragma unroll
      for (int j = 0; j < CH; ++j)
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int64_t i = tile0 + (int64_t)((warp * CH + j) * 32 + lane) * E + k;
          v[j][k] = i < p.n ? p.in[i] : T(0);
        }
    }

    // 2. in-chunk scans, then row-by-row warp scans of the chunk totals
    T off[CH];
    T running = T(0);
#pragma unroll
    for (int j = 0; j < CH; ++j) {
#pragma unroll
      for (int k = 1; k < E; ++k) v[j][k] = e_add(v[j][k], v[j][k - 1]);
      const T tot = v[j][E - 1];
      T s = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s = e_add(s, u);
      }
      off[j] = e_add(running, e_sub(s, tot));
      running = e_add(running, __shfl_sync(0xffffffffu, s, 31));
    }
    if (lane == 0) s_warp[buf][warp] = running;
    __syncthreads();  // [A] stage data consumed into registers; warp totals visible
    if (threadIdx.x == producer) refill(stage);
    if (warp == 0) {
      const T mine = lane < WARPS ? s_warp[buf][lane] : T(0);
      T w = mine;
#pragma unroll
      for (int o = 1; o < WARPS; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w = e_add(w, u);
      }
      const T block_total = __shfl_sync(0xffffffffu, w, WARPS - 1);
      T prefix;
      if (tile == 0) {
        prefix = T(0);
        if (lane == 0)
          for (int64_t c = 0; c < p.carry_count; ++c) prefix = e_add(prefix, p.carry[c]);
        prefix = __shfl_sync(0xffffffffu, prefix, 0);
        if (lane == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, e_add(prefix, block_total));
      } else {
        if (lane == 0) p.status.publish(tile, epoch, FLAG_AGGREGATE, block_total);
        prefix = look_back<T, DEPTH, 0>(p.status, tile, epoch);
        if (lane == 0) p.status.publish(tile, epoch, FLAG_INCLUSIVE, e_add(prefix, block_total));
      }
      if (lane < WARPS) s_warp[buf][lane] = e_add(prefix, e_sub(w, mine));  // warp's exclusive prefix
    }
    __syncthreads();  // [B] per-warp exclusive prefixes ready
    const T wbase = s_warp[buf][warp];

    // 3. add prefixes and store (each STG.128 of a warp covers 512 bytes)
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const T cb = e_add(wbase, off[j]);
      T o[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if constexpr (EXCLUSIVE) o[k] = k == 0 ? cb : e_add(cb, v[j][k - 1]);
        else o[k] = e_add(cb, v[j][k]);
      }
      const int64_t i = tile0 + (int64_t)((warp * CH + j) * 32 + lane) * E;
      if (full) {
        stg128(p.out + i, Chunk<T>::pack(o));
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (i + k < p.n) p.out[i + k] = o[k];
      }
    }
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1u;
    }
  }
}


// ===========================================================================
// Shared-memory-staged variant (one super-tile per CTA, dynamic tile id).
// The whole super-tile (NSUB sub-tiles of BLOCK*CH*16 bytes) is fetched with
// bulk TMA copies into shared memory — no registers are held while the data
// is in flight, so 2-3 CTAs per SM keep >= 128 KB of HBM reads outstanding
// per SM.  The CTA then (1) reduces the super-tile from shared memory and
// publishes its AGGREGATE at once, (2) looks back, (3) scans the sub-tiles
// from shared memory in order and stores with 128-bit coalesced stores.
// ===========================================================================
template <typename T, int BLOCK, int CH, int NSUB, int DEPTH, bool EXCLUSIVE>
__global__ void __launch_bounds__(BLOCK) scan_smem_kernel(ScanArgs<T> p) {
  using namespace tma;
  constexpr int WARPS = BLOCK / 32;
  constexpr int E = Chunk<T>::E;
  constexpr int SUB_BYTES = BLOCK * CH * 16;
  constexpr int TILE_BYTES = SUB_BYTES * NSUB;
  constexpr int64_t SUB = SUB_BYTES / (int)sizeof(T);
  constexpr int64_t TILE = TILE_BYTES / (int)sizeof(T);
  extern __shared__ __align__(128) uint8_t stage[];
  __shared__ uint64_t full_bar;
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ T s_warp[2][WARPS];
  __shared__ T s_red[WARPS];
  __shared__ T s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    mbar_init(&full_bar, 1);
    fence_mbar_init();
    const unsigned long long old = atomicAdd(p.ticket, 1ull);
    const uint32_t t = (uint32_t)old, e = (uint32_t)(old >> 32) & EPOCH_MASK;
    if ((int64_t)t == p.num_tiles - 1) *p.ticket = (unsigned long long)((e + 1u) & EPOCH_MASK) << 32;
    s_tile = t;
    s_epoch = e;
    const int64_t t0 = (int64_t)t * TILE;
    if (t0 + TILE <= p.n) {
      mbar_arrive_expect_tx(&full_bar, TILE_BYTES);
#pragma unroll
      for (int k = 0; k < NSUB; ++k) bulk_load(stage + k * SUB_BYTES, p.in + t0 + k * SUB, SUB_BYTES, &full_bar);
    } else {
      mbar_arrive(&full_bar);
    }
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const uint32_t epoch = s_epoch;
  const int64_t tile0 = tile * TILE;
  const bool full = tile0 + TILE <= p.n;
  mbar_wait(&full_bar, 0);

  auto load_chunk = [&](int sub, int j, T (&v)[E]) {
    const int c = (warp * CH + j) * 32 + lane;  // chunk index inside the sub-tile
    if (full) {
      Chunk<T>::unpack(lds128(stage + sub * SUB_BYTES + c * 16), v);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int64_t i = tile0 + sub * SUB + (int64_t)c * E + k;
        v[k] = i < p.n ? p.in[i] : T(0);
      }
    }
  };

  // 1. super-tile aggregate -> publish immediately (before any look-back)
  T acc = T(0);
#pragma unroll
  for (int sub = 0; sub < NSUB; ++sub)
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      T v[E];
      load_chunk(sub, j, v);
#pragma unroll
      for (int k = 0; k < E; ++k) acc = e_add(acc, v[k]);
    }
  acc = warp_sum<T>(acc);
  if (lane == 0) s_red[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < WARPS ? s_red[lane] : T(0);
    const T total = warp_sum<T>(w);
    T prefix;
    if (tile == 0) {
      prefix = T(0);
      if (lane == 0)
        for (int64_t c = 0; c < p.carry_count; ++c) prefix = e_add(prefix, p.carry[c]);
      prefix = __shfl_sync(0xffffffffu, prefix, 0);
      if (lane == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, e_add(prefix, total));
    } else {
      if (lane == 0) p.status.publish(tile, epoch, FLAG_AGGREGATE, total);
      prefix = look_back<T, DEPTH, 0>(p.status, tile, epoch);
      if (lane == 0) p.status.publish(tile, epoch, FLAG_INCLUSIVE, e_add(prefix, total));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  T carry = s_prefix;  // block-uniform running prefix across sub-tiles

  // 2. scan the sub-tiles in order
#pragma unroll 1
  for (int sub = 0; sub < NSUB; ++sub) {
    const int buf = sub & 1;
    T v[CH][E];
#pragma unroll
    for (int j = 0; j < CH; ++j) load_chunk(sub, j, v[j]);
    T off[CH];
    T running = T(0);
#pragma unroll
    for (int j = 0; j < CH; ++j) {
#pragma unroll
      for (int k = 1; k < E; ++k) v[j][k] = e_add(v[j][k], v[j][k - 1]);
      const T tot = v[j][E - 1];
      T s = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s = e_add(s, u);
      }
      off[j] = e_add(running, e_sub(s, tot));
      running = e_add(running, __shfl_sync(0xffffffffu, s, 31));
    }
    if (lane == 0) s_warp[buf][warp] = running;
    __syncthreads();
    T wex = T(0), sub_total = T(0);
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const T tw = s_warp[buf][w];
      if (w < warp) wex = e_add(wex, tw);
      sub_total = e_add(sub_total, tw);
    }
    const T wbase = e_add(carry, wex);
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const T cb = e_add(wbase, off[j]);
      T o[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if constexpr (EXCLUSIVE) o[k] = k == 0 ? cb : e_add(cb, v[j][k - 1]);
        else o[k] = e_add(cb, v[j][k]);
      }
      const int64_t i = tile0 + sub * SUB + (int64_t)((warp * CH + j) * 32 + lane) * E;
      if (full) {
        stg128(p.out + i, Chunk<T>::pack(o));
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (i + k < p.n) p.out[i + k] = o[k];
      }
    }
    carry = e_add(carry, sub_total);
  }
}


// ===========================================================================
// Warp-specialized persistent variant: the look-back never stalls HBM reads.
//   warp 0 (producer): claims tiles from the ticket and starts a bulk TMA copy
//                      of each into a free ring stage (mbarriers full/empty);
//   warp 1 (aggregator): as soon as a stage lands, reduces it from shared
//                      memory (one 512-byte row per LDS.128, C independent
//                      per-slice accumulators) and publishes the tile's
//                      AGGREGATE plus the exclusive offset of every slice;
//   warps 2..2+NL-1 (look-back): take the uses round-robin, walk back over
//                      predecessors (whose aggregates appear as soon as THEIR
//                      data lands) and publish INCLUSIVE;
//   C consumer warps: scan their CH rows of the stage, free the stage, wait
//                      for the tile prefix, add it and store (STG.128 rows).
// Stage data moves through full/empty mbarriers.  The per-use results of the
// aggregator and the look-back warps go through SLOTS = 2*STAGES slots tagged
// with the use number (no phase aliasing when a role runs ahead: the ring
// bounds how far any writer can get ahead of the slowest reader).
// ===========================================================================
__device__ __forceinline__ uint32_t ld_volatile_shared(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(tma::smem_u32(p)) : "memory");
  return v;
}
// Spin until *flag == want (written by another warp of this CTA); trap after 10 s.
__device__ __forceinline__ void wait_flag(const uint32_t *flag, uint32_t want) {
  if (ld_volatile_shared(flag) == want) {
    __threadfence_block();
    return;
  }
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (ld_volatile_shared(flag) != want) {
    __nanosleep(20);
    if ((++spins & 1023u) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 10000000000ull) __trap();
    }
  }
  __threadfence_block();
}

template <typename T, int C, int CH, int STAGES, int DEPTH, int NL, bool EXCLUSIVE>
__global__ void __launch_bounds__((2 + NL + C) * 32) scan_ws_kernel(ScanArgs<T> p) {
  using namespace tma;
  constexpr int E = Chunk<T>::E;
  constexpr int ROW_BYTES = 512;  // one warp-wide LDS.128 / STG.128
  constexpr int SLICE_BYTES = CH * ROW_BYTES;
  constexpr int TILE_BYTES = C * SLICE_BYTES;
  constexpr int64_t TILE = TILE_BYTES / (int)sizeof(T);
  constexpr int FIRST_CONSUMER = 2 + NL;
  constexpr int SLOTS = 2 * STAGES;
  static_assert(NL <= STAGES, "look-back warps must not outnumber stages");
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ long long stage_tile[STAGES];
  __shared__ T slice_off[SLOTS][C];
  __shared__ T tile_total[SLOTS];
  __shared__ T tile_prefix[SLOTS];
  __shared__ long long slot_tile[SLOTS];
  __shared__ uint32_t agg_done[SLOTS], pref_done[SLOTS];  // use number + 1 when ready
  __shared__ uint32_t s_epoch;
  __shared__ uint32_t s_end;  // use number at which the producer ran out of tiles
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], C + 1);
    }
    for (int s = 0; s < SLOTS; ++s) agg_done[s] = pref_done[s] = 0u;
    s_end = 0xffffffffu;
    fence_mbar_init();
  }
  __syncthreads();

  auto read_chunk = [&](int stage, long long tile, bool full, int row, T (&v)[E]) {
    if (full) {
      Chunk<T>::unpack(lds128(ring + (size_t)stage * TILE_BYTES + row * ROW_BYTES + lane * 16), v);
    } else {
      const int64_t i0 = (int64_t)tile * TILE + (int64_t)(row * 32 + lane) * E;
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = i0 + k < p.n ? p.in[i0 + k] : T(0);
    }
  };
  auto carry_in = [&]() {
    T c = T(0);
    for (int64_t k = 0; k < p.carry_count; ++k) c = e_add(c, p.carry[k]);
    return c;
  };

  if (warp == 0) {
    // ---------------- producer
    if (lane != 0) return;
    const int64_t last_claim = p.num_tiles + (int64_t)gridDim.x - 1;
    for (uint32_t k = 0;; ++k) {
      const int s = (int)(k % STAGES);
      const uint32_t use = k / STAGES;
      if (use > 0) mbar_wait(&empty_bar[s], (use - 1) & 1u);
      const unsigned long long old = atomicAdd(p.ticket, 1ull);
      const int64_t t = (int64_t)(uint32_t)old;
      const uint32_t e = (uint32_t)(old >> 32) & EPOCH_MASK;
      s_epoch = e;
      if (t == last_claim) *p.ticket = (unsigned long long)((e + 1u) & EPOCH_MASK) << 32;
      if (t < p.num_tiles) {
        stage_tile[s] = t;
        if (p.trace) p.trace[t * 8 + 0] = globaltimer_ns();
        if ((t + 1) * TILE <= p.n) {
          fence_proxy_async();
          mbar_arrive_expect_tx(&full_bar[s], TILE_BYTES);
          bulk_load(ring + (size_t)s * TILE_BYTES, p.in + t * TILE, TILE_BYTES, &full_bar[s]);
        } else {
          mbar_arrive(&full_bar[s]);  // ragged last tile: readers use global memory
        }
      } else {
        stage_tile[s] = -1;  // no more work: every role stops at this use
        mbar_arrive(&full_bar[s]);
        return;
      }
    }
  } else if (warp == 1) {
    // ---------------- aggregator
    for (uint32_t k = 0;; ++k) {
      const int s = (int)(k % STAGES);
      const int slot = (int)(k % SLOTS);
      mbar_wait(&full_bar[s], (k / STAGES) & 1u);
      const long long t = stage_tile[s];
      if (t < 0) {
        if (lane == 0) {
          s_end = k;
          __threadfence_block();
          for (uint32_t r = 0; r < NL; ++r) ((volatile uint32_t *)agg_done)[(k + r) % SLOTS] = k + r + 1;
        }
        return;
      }
      const uint32_t epoch = s_epoch;
      const bool full = (int64_t)(t + 1) * TILE <= p.n;
      if (p.trace && lane == 0) p.trace[t * 8 + 1] = globaltimer_ns();
      T acc[C];
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = T(0);
#pragma unroll 2
      for (int j = 0; j < CH; ++j) {
#pragma unroll
        for (int c = 0; c < C; ++c) {  // C independent rows in flight
          T v[E];
          read_chunk(s, t, full, c * CH + j, v);
          T r = v[0];
#pragma unroll
          for (int q = 1; q < E; ++q) r = e_add(r, v[q]);
          acc[c] = e_add(acc[c], r);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);  // stage no longer read by this warp
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = e_add(acc[c], __shfl_xor_sync(0xffffffffu, acc[c], o));
      if (lane == 0) {
        T run = T(0);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          slice_off[slot][c] = run;
          run = e_add(run, acc[c]);
        }
        tile_total[slot] = run;
        slot_tile[slot] = t;
        if (t == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, e_add(carry_in(), run));
        else p.status.publish(t, epoch, FLAG_AGGREGATE, run);
        if (p.trace) p.trace[t * 8 + 2] = globaltimer_ns();
        __threadfence_block();
        ((volatile uint32_t *)agg_done)[slot] = k + 1;
      }
      __syncwarp();
    }
  } else if (warp < FIRST_CONSUMER) {
    // ---------------- look-back (NL warps, uses round-robin)
    for (uint32_t k = (uint32_t)(warp - 2);; k += NL) {
      const int slot = (int)(k % SLOTS);
      wait_flag(&agg_done[slot], k + 1);
      if (k >= ld_volatile_shared(&s_end)) return;
      const long long t = slot_tile[slot];
      const uint32_t epoch = s_epoch;
      if (p.trace && lane == 0) p.trace[t * 8 + 3] = globaltimer_ns();
      T prefix;
      if (t == 0) {
        prefix = lane == 0 ? carry_in() : T(0);
        prefix = __shfl_sync(0xffffffffu, prefix, 0);
      } else {
        prefix = look_back<T, DEPTH, 0>(p.status, t, epoch);
        if (lane == 0) p.status.publish(t, epoch, FLAG_INCLUSIVE, e_add(prefix, tile_total[slot]));
      }
      if (lane == 0) {
        tile_prefix[slot] = prefix;
        if (p.trace) p.trace[t * 8 + 4] = globaltimer_ns();
        __threadfence_block();
        ((volatile uint32_t *)pref_done)[slot] = k + 1;
      }
      __syncwarp();
    }
  } else {
    // ---------------- consumers
    const int c = warp - FIRST_CONSUMER;
    for (uint32_t k = 0;; ++k) {
      const int s = (int)(k % STAGES);
      const int slot = (int)(k % SLOTS);
      mbar_wait(&full_bar[s], (k / STAGES) & 1u);
      const long long t = stage_tile[s];
      if (t < 0) return;
      const bool full = (int64_t)(t + 1) * TILE <= p.n;
      T v[CH][E];
#pragma unroll
      for (int j = 0; j < CH; ++j) read_chunk(s, t, full, c * CH + j, v[j]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);  // stage bytes are in registers now
      T off[CH];
      T running = T(0);
#pragma unroll
      for (int j = 0; j < CH; ++j) {
#pragma unroll
        for (int q = 1; q < E; ++q) v[j][q] = e_add(v[j][q], v[j][q - 1]);
        const T tot = v[j][E - 1];
        T x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const T u = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x = e_add(x, u);
        }
        off[j] = e_add(running, e_sub(x, tot));
        running = e_add(running, __shfl_sync(0xffffffffu, x, 31));
      }
      if (p.trace && c == 0 && lane == 0) p.trace[t * 8 + 5] = globaltimer_ns();
      wait_flag(&pref_done[slot], k + 1);
      const T base = e_add(tile_prefix[slot], slice_off[slot][c]);
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const T cb = e_add(base, off[j]);
        T o[E];
#pragma unroll
        for (int q = 0; q < E; ++q) {
          if constexpr (EXCLUSIVE) o[q] = q == 0 ? cb : e_add(cb, v[j][q - 1]);
          else o[q] = e_add(cb, v[j][q]);
        }
        const int64_t i = (int64_t)t * TILE + (int64_t)((c * CH + j) * 32 + lane) * E;
        if (full) {
          stg128(p.out + i, Chunk<T>::pack(o));
        } else {
#pragma unroll
          for (int q = 0; q < E; ++q)
            if (i + q < p.n) p.out[i + q] = o[q];
        }
      }
      if (p.trace && c == 0 && lane == 0) p.trace[t * 8 + 6] = globaltimer_ns();
    }
  }
}


// ===========================================================================
// Two-touch variant (reduce then scan, one launch, the super-tile re-read
// from L2).  One CTA per super-tile (dynamic id); warp w owns ROWS
// consecutive 512-byte rows (its slice):
//   phase 1  stream the slice from HBM (UNROLL rows in flight per warp,
//            L2 evict_last) and sum it; the block turns the slice sums into
//            slice offsets and the super-tile AGGREGATE, published at once;
//   phase 2  warp 0 looks back for the super-tile prefix;
//   phase 3  every warp re-reads its slice (now L2-resident, evict_first),
//            scans it row by row and stores (STG.128, 512 B per warp).
// HBM traffic stays 1 read + 1 write per element when the super-tiles in
// flight fit in L2; the aggregate is published after a long streaming phase
// whose duration varies little between CTAs, so look-back waits are short.
// ===========================================================================
namespace l2 {
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <bool NC>
__device__ __forceinline__ uint4 ldg128_hint(const void *p, uint64_t pol) {
  uint4 v;
  if constexpr (NC)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol)
                 : "memory");
  return v;
}
template <bool NC>
__device__ __forceinline__ uint4 ldg128(const void *p) {
  uint4 v;
  if constexpr (NC)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
  return v;
}
__device__ __forceinline__ void stg128_hint(void *p, const uint4 &v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
}  // namespace l2

// STAGE_SMEM: phase 1 also parks every row in shared memory (dynamic smem of
// WARPS*ROWS*512 bytes) and phase 3 reads it from there instead of L2.
// EARLY: warps 1..WARPS-1 load and locally scan their first UNROLL rows of
// phase 3 while warp 0 is still in the look-back.
template <typename T, int WARPS, int ROWS, int UNROLL, int DEPTH, bool HINTS, bool NC, bool EXCLUSIVE,
          bool STAGE_SMEM = false, bool EARLY = false, int MINB = 1>
__global__ void __launch_bounds__(WARPS * 32, MINB) scan_l2_kernel(ScanArgs<T> p) {
  extern __shared__ __align__(128) uint8_t park[];
  using namespace tma;
  constexpr int E = Chunk<T>::E;
  constexpr int ROW = 32 * E;                      // elements per 512-byte row
  constexpr int64_t TILE = (int64_t)WARPS * ROWS * ROW;
  static_assert(ROWS % UNROLL == 0, "ROWS must be a multiple of UNROLL");
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ T s_slice[WARPS];
  __shared__ T s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    const unsigned long long old = atomicAdd(p.ticket, 1ull);
    const uint32_t t = (uint32_t)old, e = (uint32_t)(old >> 32) & EPOCH_MASK;
    if ((int64_t)t == p.num_tiles - 1) *p.ticket = (unsigned long long)((e + 1u) & EPOCH_MASK) << 32;
    s_tile = t;
    s_epoch = e;
    if (p.trace) p.trace[(int64_t)t * 8 + 0] = globaltimer_ns();
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const uint32_t epoch = s_epoch;
  const int64_t slice0 = tile * TILE + (int64_t)warp * ROWS * ROW;  // first element of my slice
  const bool full = tile * TILE + TILE <= p.n;
  const uint64_t keep = HINTS ? l2::policy_evict_last() : 0;
  const uint64_t drop = HINTS ? l2::policy_evict_first() : 0;

  auto load_row = [&](int r, uint64_t pol, T (&v)[E]) {
    const int64_t i = slice0 + (int64_t)r * ROW + lane * E;
    if (full) {
      uint4 raw;
      if constexpr (HINTS) raw = l2::ldg128_hint<NC>(p.in + i, pol);
      else raw = l2::ldg128<NC>(p.in + i);
      Chunk<T>::unpack(raw, v);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = i + k < p.n ? p.in[i + k] : T(0);
    }
  };

  uint8_t *my_park = park + ((size_t)warp * ROWS * 512 + lane * 16);

  // phase 1: slice sums
  T acc = T(0);
#pragma unroll 1
  for (int r0 = 0; r0 < ROWS; r0 += UNROLL) {
    T v[UNROLL][E];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) load_row(r0 + u, keep, v[u]);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if constexpr (STAGE_SMEM) {
        const uint4 raw = Chunk<T>::pack(v[u]);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(my_park + (r0 + u) * 512)), "r"(raw.x),
                     "r"(raw.y), "r"(raw.z), "r"(raw.w)
                     : "memory");
      }
#pragma unroll
      for (int k = 0; k < E; ++k) acc = e_add(acc, v[u][k]);
    }
  }
  acc = warp_sum<T>(acc);
  if (lane == 0) s_slice[warp] = acc;
  __syncthreads();

  // phase 2: slice offsets, aggregate, look-back (warp 0)
  if (warp == 0) {
    const T mine = lane < WARPS ? s_slice[lane] : T(0);
    T w = mine;
#pragma unroll
    for (int o = 1; o < WARPS; o <<= 1) {
      const T u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = e_add(w, u);
    }
    const T total = __shfl_sync(0xffffffffu, w, WARPS - 1);
    T prefix;
    if (p.trace && lane == 0) p.trace[tile * 8 + 1] = globaltimer_ns();
    if (tile == 0) {
      prefix = T(0);
      if (lane == 0)
        for (int64_t c = 0; c < p.carry_count; ++c) prefix = e_add(prefix, p.carry[c]);
      prefix = __shfl_sync(0xffffffffu, prefix, 0);
      if (lane == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, e_add(prefix, total));
    } else {
      if (lane == 0) p.status.publish(tile, epoch, FLAG_AGGREGATE, total);
      prefix = look_back<T, DEPTH, 0>(p.status, tile, epoch);
      if (lane == 0) p.status.publish(tile, epoch, FLAG_INCLUSIVE, e_add(prefix, total));
    }
    if (p.trace && lane == 0) p.trace[tile * 8 + 2] = globaltimer_ns();
    if (lane < WARPS) s_slice[lane] = e_add(prefix, e_sub(w, mine));  // exclusive prefix of slice `lane`
  }
  // phase 3: re-read (L2 or the parked copy), scan row by row, store.
  // load_local: rows [r0, r0+UNROLL) into registers, in-row scans, and each
  // row's exclusive offset relative to the chunk start (off) + chunk total.
  auto load_local = [&](int r0, T (&v)[UNROLL][E], T (&off)[UNROLL], T &ctot) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if constexpr (STAGE_SMEM) Chunk<T>::unpack(lds128(my_park + (r0 + u) * 512), v[u]);
      else load_row(r0 + u, drop, v[u]);
    }
    ctot = T(0);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
#pragma unroll
      for (int k = 1; k < E; ++k) v[u][k] = e_add(v[u][k], v[u][k - 1]);
      const T tot = v[u][E - 1];
      T x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = e_add(x, y);
      }
      off[u] = e_add(ctot, e_sub(x, tot));
      ctot = e_add(ctot, __shfl_sync(0xffffffffu, x, 31));
    }
  };
  auto store_chunk = [&](int r0, const T (&v)[UNROLL][E], const T (&off)[UNROLL], T base) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const T cb = e_add(base, off[u]);
      T o[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if constexpr (EXCLUSIVE) o[k] = k == 0 ? cb : e_add(cb, v[u][k - 1]);
        else o[k] = e_add(cb, v[u][k]);
      }
      const int64_t i = slice0 + (int64_t)(r0 + u) * ROW + lane * E;
      if (full) {
        if constexpr (HINTS) l2::stg128_hint(p.out + i, Chunk<T>::pack(o), drop);
        else stg128(p.out + i, Chunk<T>::pack(o));
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (i + k < p.n) p.out[i + k] = o[k];
      }
    }
  };
  T v0[UNROLL][E], off0[UNROLL], ctot0;
  const bool early = EARLY && warp != 0;
  if (early) load_local(0, v0, off0, ctot0);
  __syncthreads();
  T base = s_slice[warp];
  if (!early) load_local(0, v0, off0, ctot0);
  store_chunk(0, v0, off0, base);
  base = e_add(base, ctot0);
#pragma unroll 1
  for (int r0 = UNROLL; r0 < ROWS; r0 += UNROLL) {
    T v[UNROLL][E], off[UNROLL], ctot;
    load_local(r0, v, off, ctot);
    store_chunk(r0, v, off, base);
    base = e_add(base, ctot);
  }
  if (p.trace && threadIdx.x == 0) p.trace[tile * 8 + 3] = globaltimer_ns();
}

// ===========================================================================
// Pipelined two-touch variant (persistent, warp-specialized, one CTA per SM).
//   RW reader warps   : stream super-tile k+1 from HBM and sum its RW slices
//                       (phase 1), claiming the next id one iteration ahead;
//   1 look-back warp  : turns the slice sums of k+1 into the AGGREGATE,
//                       publishes it, looks back, publishes INCLUSIVE and the
//                       per-slice exclusive prefixes;
//   RW writer warps   : re-read super-tile k from L2, scan it and store
//                       (phase 3).
// Phase 1 of one super-tile, the look-back of the next and phase 3 of the
// previous overlap inside every SM, so HBM sees reads and writes all the
// time and look-back latency hides behind the writers.  Hand-off through two
// shared-memory buffers guarded by sequence flags.
// ===========================================================================
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void st_volatile_shared(uint32_t *p, uint32_t v) {
  asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(tma::smem_u32(p)), "r"(v) : "memory");
}

template <typename T, int RW, int ROWS, int RU, int WU, int DEPTH, bool NC, bool EXCLUSIVE>
__global__ void __launch_bounds__((2 * RW + 1) * 32, 1) scan_pipe_kernel(ScanArgs<T> p) {
  using namespace tma;
  constexpr int E = Chunk<T>::E;
  constexpr int ROW = 32 * E;  // elements per 512-byte row
  constexpr int64_t SLICE = (int64_t)ROWS * ROW;
  constexpr int64_t TILE = (int64_t)RW * SLICE;
  static_assert(ROWS % RU == 0 && ROWS % WU == 0, "ROWS must be a multiple of the unrolls");
  static_assert(RW <= 32, "slice sums are scanned by one warp");
  __shared__ long long s_tile[2];
  __shared__ T s_sums[2][RW];
  __shared__ T s_off[2][RW];
  __shared__ uint32_t sums_ready[2], prefix_ready[2], buf_free[2];
  __shared__ uint32_t s_epoch;
  __shared__ long long s_next;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t last_claim = p.num_tiles + (int64_t)gridDim.x - 1;

  if (threadIdx.x == 0) {
    sums_ready[0] = sums_ready[1] = prefix_ready[0] = prefix_ready[1] = buf_free[0] = buf_free[1] = 0u;
  }
  __syncthreads();

  auto load_row = [&](long long tile, int slice, int r, uint64_t pol, bool full, T (&v)[E]) {
    const int64_t i = (int64_t)tile * TILE + slice * SLICE + (int64_t)r * ROW + lane * E;
    if (full) {
      Chunk<T>::unpack(l2::ldg128_hint<NC>(p.in + i, pol), v);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = i + k < p.n ? p.in[i + k] : T(0);
    }
  };
  // one claim: returns the tile id or -1; resets the ticket on the globally last claim
  auto claim = [&]() -> long long {
    const unsigned long long old = atomicAdd(p.ticket, 1ull);
    const int64_t t = (int64_t)(uint32_t)old;
    const uint32_t e = (uint32_t)(old >> 32) & EPOCH_MASK;
    s_epoch = e;
    if (t == last_claim) *p.ticket = (unsigned long long)((e + 1u) & EPOCH_MASK) << 32;
    return t < p.num_tiles ? (long long)t : -1ll;
  };

  if (warp < RW) {
    // ------------------------------------------------ readers (phase 1)
    const uint64_t keep = l2::policy_evict_last();
    long long next = -1;
    if (threadIdx.x == 0) next = claim();
    for (uint32_t k = 0;; ++k) {
      const int buf = k & 1;
      if (k >= 2) wait_flag(&buf_free[buf], k - 1);
      if (threadIdx.x == 0) {
        s_tile[buf] = next;
        // claim the following id now; its latency overlaps this phase
        s_next = next >= 0 ? claim() : -1ll;
      }
      named_bar(1, RW * 32);
      const long long t = s_tile[buf];
      if (threadIdx.x == 0) next = s_next;
      if (t < 0) {
        if (threadIdx.x == 0) {
          __threadfence_block();
          st_volatile_shared(&sums_ready[buf], k + 1);
        }
        return;
      }
      const bool full = (int64_t)(t + 1) * TILE <= p.n;
      T acc = T(0);
#pragma unroll 1
      for (int r0 = 0; r0 < ROWS; r0 += RU) {
        T v[RU][E];
#pragma unroll
        for (int u = 0; u < RU; ++u) load_row(t, warp, r0 + u, keep, full, v[u]);
#pragma unroll
        for (int u = 0; u < RU; ++u)
#pragma unroll
          for (int q = 0; q < E; ++q) acc = e_add(acc, v[u][q]);
      }
      acc = warp_sum<T>(acc);
      if (lane == 0) s_sums[buf][warp] = acc;
      named_bar(1, RW * 32);
      if (threadIdx.x == 0) {
        __threadfence_block();
        st_volatile_shared(&sums_ready[buf], k + 1);
      }
    }
  } else if (warp == RW) {
    // ------------------------------------------------ look-back warp
    for (uint32_t k = 0;; ++k) {
      const int buf = k & 1;
      wait_flag(&sums_ready[buf], k + 1);
      const long long t = s_tile[buf];
      if (t < 0) {
        if (lane == 0) {
          __threadfence_block();
          st_volatile_shared(&prefix_ready[buf], k + 1);
        }
        return;
      }
      const uint32_t epoch = s_epoch;
      const T mine = lane < RW ? s_sums[buf][lane] : T(0);
      T w = mine;
#pragma unroll
      for (int o = 1; o < RW; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w = e_add(w, u);
      }
      const T total = __shfl_sync(0xffffffffu, w, RW - 1);
      T prefix;
      if (t == 0) {
        prefix = T(0);
        if (lane == 0)
          for (int64_t c = 0; c < p.carry_count; ++c) prefix = e_add(prefix, p.carry[c]);
        prefix = __shfl_sync(0xffffffffu, prefix, 0);
        if (lane == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, e_add(prefix, total));
      } else {
        if (lane == 0) p.status.publish(t, epoch, FLAG_AGGREGATE, total);
        prefix = look_back<T, DEPTH, 0>(p.status, t, epoch);
        if (lane == 0) p.status.publish(t, epoch, FLAG_INCLUSIVE, e_add(prefix, total));
      }
      if (lane < RW) s_off[buf][lane] = e_add(prefix, e_sub(w, mine));
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        st_volatile_shared(&prefix_ready[buf], k + 1);
      }
    }
  } else {
    // ------------------------------------------------ writers (phase 3)
    const int slice = warp - RW - 1;
    const uint64_t drop = l2::policy_evict_first();
    for (uint32_t k = 0;; ++k) {
      const int buf = k & 1;
      wait_flag(&prefix_ready[buf], k + 1);
      const long long t = s_tile[buf];
      if (t < 0) return;
      const bool full = (int64_t)(t + 1) * TILE <= p.n;
      T base = s_off[buf][slice];
#pragma unroll 1
      for (int r0 = 0; r0 < ROWS; r0 += WU) {
        T v[WU][E];
#pragma unroll
        for (int u = 0; u < WU; ++u) load_row(t, slice, r0 + u, drop, full, v[u]);
#pragma unroll
        for (int u = 0; u < WU; ++u) {
#pragma unroll
          for (int q = 1; q < E; ++q) v[u][q] = e_add(v[u][q], v[u][q - 1]);
          const T tot = v[u][E - 1];
          T x = tot;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = e_add(x, y);
          }
          const T cb = e_add(base, e_sub(x, tot));
          base = e_add(base, __shfl_sync(0xffffffffu, x, 31));
          T o[E];
#pragma unroll
          for (int q = 0; q < E; ++q) {
            if constexpr (EXCLUSIVE) o[q] = q == 0 ? cb : e_add(cb, v[u][q - 1]);
            else o[q] = e_add(cb, v[u][q]);
          }
          const int64_t i = (int64_t)t * TILE + slice * SLICE + (int64_t)(r0 + u) * ROW + lane * E;
          if (full) {
            l2::stg128_hint(p.out + i, Chunk<T>::pack(o), drop);
          } else {
#pragma unroll
            for (int q = 0; q < E; ++q)
              if (i + q < p.n) p.out[i + q] = o[q];
          }
        }
      }
      named_bar(2, RW * 32);
      if (slice == 0 && lane == 0) {
        __threadfence_block();
        st_volatile_shared(&buf_free[buf], k + 1);
      }
    }
  }
}

}  // namespace scan_lab_old
}  // namespace ga
