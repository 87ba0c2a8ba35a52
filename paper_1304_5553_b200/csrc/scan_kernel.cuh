// scan_kernel.cuh — the product scan kernels (see scan.cu for the algorithm
// and its citations), generic over the scan expression OP ∈ {SUM, MAX, MIN}
// (P:496-499 with the reduction expressions of P:479-485) and the element
// type T ∈ {int32, int64, float, double}.
//
//   scan_l2_kernel  the tuned two-touch super-tile kernel (16-byte aligned
//                   arrays): phase 1 streams and folds the super-tile,
//                   publishes its AGGREGATE, warp 0 looks back, phase 3
//                   re-reads it from L2, scans and stores.
//   scan_reg_kernel the fallback for arrays that are not 16-byte aligned:
//                   one register tile per CTA, scalar loads.
// Both share the decoupled look-back machinery below.  The alternatives
// measured while tuning are described in DESIGN.md §6 (tuning history).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "ga_device.cuh"

namespace ga {
namespace scan_detail {

constexpr uint32_t FLAG_INVALID = 0, FLAG_AGGREGATE = 1, FLAG_INCLUSIVE = 2;
constexpr uint32_t EPOCH_MASK = (1u << 30) - 1;
// Workspace header: one 64-bit ticket word {epoch:32 | tile counter:32} in its
// own 256-byte block; per-tile status follows.
constexpr size_t HEADER = 256;

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// 32-bit payload of a 4-byte element (bit pattern, any type).
template <typename T>
__device__ __forceinline__ uint32_t to_bits32(T v) {
  if constexpr (std::is_same<T, float>::value) return __float_as_uint(v);
  else return (uint32_t)v;
}
template <typename T>
__device__ __forceinline__ T from_bits32(uint32_t b) {
  if constexpr (std::is_same<T, float>::value) return __uint_as_float(b);
  else return (T)b;
}
// 64-bit payload of an 8-byte element.
template <typename T>
__device__ __forceinline__ uint64_t to_bits64(T v) {
  if constexpr (std::is_same<T, double>::value) return (uint64_t)__double_as_longlong(v);
  else return (uint64_t)v;
}
template <typename T>
__device__ __forceinline__ T from_bits64(uint64_t b) {
  if constexpr (std::is_same<T, double>::value) return __longlong_as_double((long long)b);
  else return (T)b;
}

// Look-back status of one tile.  Every 64-bit word of the status region
// carries a tag (epoch:30 | flag:2) in its high half and 32 payload bits in
// its low half, whatever the element size, at a per-tile stride of
// sizeof(T) * 2 bytes from the same base:
//  4-byte T: one word   tag << 32 | bits(value);
//  8-byte T: two words  tag << 32 | lo32(value),  tag << 32 | hi32(value).
// Each word is written and read with single-copy-atomic 64-bit accesses; a
// status is valid for the current call when every word carries the call's
// epoch and the same flag (an 8-byte status caught between its AGGREGATE
// and INCLUSIVE publications shows two flags and is re-read).  Because the
// region never holds an untagged word, a workspace reused across element
// sizes, tile counts and shapes can only show tags of earlier epochs, which
// never match (the layout-independent status).
template <typename T, int SZ = sizeof(T)>
struct Status;

__device__ __forceinline__ uint64_t tag_word(uint32_t epoch, uint32_t flag, uint32_t payload) {
  return ((uint64_t)((epoch << 2) | flag) << 32) | payload;
}
__device__ __forceinline__ uint32_t tag_flag(uint32_t hi, uint32_t epoch) {
  return (hi >> 2) == epoch ? (hi & 3u) : FLAG_INVALID;
}

template <typename T>
struct Status<T, 4> {
  uint64_t *word;
  __device__ void publish(int64_t tile, uint32_t epoch, uint32_t flag, T v) const {
    st_relaxed_u64(word + tile, tag_word(epoch, flag, to_bits32<T>(v)));
  }
  __device__ uint32_t read(int64_t tile, uint32_t epoch, T &v) const {
    const uint64_t w = ld_relaxed_u64(word + tile);
    v = from_bits32<T>((uint32_t)w);
    return tag_flag((uint32_t)(w >> 32), epoch);
  }
};

template <typename T>
struct Status<T, 8> {
  uint64_t *word;  // two words per tile
  __device__ void publish(int64_t tile, uint32_t epoch, uint32_t flag, T v) const {
    const uint64_t b = to_bits64<T>(v);
    const uint64_t lo = tag_word(epoch, flag, (uint32_t)b), hi = tag_word(epoch, flag, (uint32_t)(b >> 32));
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(word + 2 * tile), "l"(lo), "l"(hi)
                 : "memory");
  }
  __device__ uint32_t read(int64_t tile, uint32_t epoch, T &v) const {
    uint64_t lo, hi;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(word + 2 * tile)
                 : "memory");
    const uint32_t tlo = (uint32_t)(lo >> 32), thi = (uint32_t)(hi >> 32);
    v = from_bits64<T>(((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo);
    return tlo == thi ? tag_flag(tlo, epoch) : FLAG_INVALID;
  }
};

// Tin: the input element type; T: the scan (accumulator, output, status,
// carry) type — equal, or a widening int32 -> int64 / float -> double.
template <typename T, typename Tin = T>
struct ScanArgs {
  int64_t n;
  int64_t num_tiles;
  const Tin *in;
  T *out;
  const T *carry;
  int64_t carry_count;
  unsigned long long *ticket;  // {epoch:32 | counter:32}
  Status<T> status;
  int64_t pf_dist;  // PF_ROWS kernels: prefetch into L2 the tile this many ids ahead (0: off)
};

// Spin until predecessor `idx` has published.  A predecessor that stays
// INVALID for 10 s means a corrupted workspace: trap instead of hanging.
template <typename T>
__device__ __forceinline__ uint32_t wait_status(const Status<T> &st, int64_t idx, uint32_t epoch, T &v) {
  uint32_t f = st.read(idx, epoch, v);
  if (f != FLAG_INVALID) return f;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while ((f = st.read(idx, epoch, v)) == FLAG_INVALID) {
    if ((++spins & 1023u) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 10000000000ull) __trap();
    }
  }
  return f;
}

// Warp 0: exclusive prefix (fold of all predecessors) of `tile`.  Each round
// reads 32*DEPTH predecessors (DEPTH independent loads per lane in flight),
// waits until all are published, and stops at the nearest INCLUSIVE.  The
// fold order within a round is the fixed xor butterfly, so integer and
// max/min results are exact; float SUM depends on which predecessors were
// INCLUSIVE at the time (R22).
template <int OP, typename T, int DEPTH>
__device__ __noinline__ T look_back(const Status<T> &st, int64_t tile, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  const T neutral = Op<OP, T>::neutral();
  T prefix = neutral;
  int64_t pred = tile - 1;
  while (true) {
    T v[DEPTH];
    uint32_t f[DEPTH];
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      const int64_t idx = pred - lane - 32 * j;  // distance 1 + lane + 32 j
      v[j] = neutral;
      f[j] = FLAG_INCLUSIVE;  // before tile 0: the neutral element
      if (idx >= 0) f[j] = st.read(idx, epoch, v[j]);
    }
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      const int64_t idx = pred - lane - 32 * j;
      if (f[j] == FLAG_INVALID) f[j] = wait_status<T>(st, idx, epoch, v[j]);
    }
    T part = neutral;
    bool done = false;
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      if (!done) {
        const uint32_t m = __ballot_sync(0xffffffffu, f[j] == FLAG_INCLUSIVE);
        if (m) {
          const int first = __ffs(m) - 1;  // nearest INCLUSIVE in this row
          part = Op<OP, T>::fold(part, lane <= first ? v[j] : neutral);
          done = true;
        } else {
          part = Op<OP, T>::fold(part, v[j]);
        }
      }
    }
    // predecessors are further back than everything folded so far
    prefix = Op<OP, T>::fold(warp_fold<OP, T>(part), prefix);
    if (done) return prefix;
    pred -= 32 * DEPTH;
  }
}

// Carry-in: fold of carry[0..carry_count) in index order (neutral if none).
template <int OP, typename T, typename Tin>
__device__ __forceinline__ T carry_in(const ScanArgs<T, Tin> &p) {
  T c = Op<OP, T>::neutral();
  for (int64_t k = 0; k < p.carry_count; ++k) c = Op<OP, T>::fold(c, p.carry[k]);
  return c;
}

// Warp-wide inclusive scan (Hillis-Steele over __shfl_up) and the matching
// exclusive value (the lane below's inclusive; the neutral for lane 0).
template <int OP, typename T>
__device__ __forceinline__ T warp_inclusive(T x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = Op<OP, T>::fold(u, x);
  }
  return x;
}
template <int OP, typename T>
__device__ __forceinline__ T warp_exclusive_of(T inclusive, int lane) {
  const T u = __shfl_up_sync(0xffffffffu, inclusive, 1);
  return lane == 0 ? Op<OP, T>::neutral() : u;
}

// ------------------------------------------------------------------ 16-byte chunks
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

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
struct Chunk<float> {
  static constexpr int E = 4;
  __device__ static void unpack(const uint4 &v, float (&e)[4]) {
    e[0] = __uint_as_float(v.x);
    e[1] = __uint_as_float(v.y);
    e[2] = __uint_as_float(v.z);
    e[3] = __uint_as_float(v.w);
  }
  __device__ static uint4 pack(const float (&e)[4]) {
    return make_uint4(__float_as_uint(e[0]), __float_as_uint(e[1]), __float_as_uint(e[2]), __float_as_uint(e[3]));
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
template <>
struct Chunk<double> {
  static constexpr int E = 2;
  __device__ static void unpack(const uint4 &v, double (&e)[2]) {
    e[0] = __hiloint2double((int)v.y, (int)v.x);
    e[1] = __hiloint2double((int)v.w, (int)v.z);
  }
  __device__ static uint4 pack(const double (&e)[2]) {
    return make_uint4((uint32_t)__double2loint(e[0]), (uint32_t)__double2hiint(e[0]), (uint32_t)__double2loint(e[1]),
                      (uint32_t)__double2hiint(e[1]));
  }
};

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
// 32 bytes per lane (a widened row: 4 int64 / double outputs per lane).
__device__ __forceinline__ void stg256_hint(void *p, const uint4 &a, const uint4 &b, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p),
               "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w), "l"(pol)
               : "memory");
}
template <bool NC>
__device__ __forceinline__ V32 ldg256_hint(const void *p, uint64_t pol) {
  V32 v;
  if constexpr (NC)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]), "=r"(v.r[6]),
                   "=r"(v.r[7])
                 : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]), "=r"(v.r[6]),
                   "=r"(v.r[7])
                 : "l"(p), "l"(pol)
                 : "memory");
  return v;
}
__device__ __forceinline__ void stg256v_hint(void *p, const V32 &v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p),
               "r"(v.r[0]), "r"(v.r[1]), "r"(v.r[2]), "r"(v.r[3]), "r"(v.r[4]), "r"(v.r[5]), "r"(v.r[6]), "r"(v.r[7]),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void stg128_hint(void *p, const uint4 &v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
}  // namespace l2

// Draw {epoch, tile id}; the CTA drawing the last id resets the counter and
// bumps the epoch (every CTA has drawn by then).
template <typename A>
__device__ __forceinline__ void draw_tile(const A &p, uint32_t &tile, uint32_t &epoch) {
  const unsigned long long old = atomicAdd(p.ticket, 1ull);
  tile = (uint32_t)old;
  epoch = (uint32_t)(old >> 32) & EPOCH_MASK;
  if ((int64_t)tile == p.num_tiles - 1) *p.ticket = (unsigned long long)((epoch + 1u) & EPOCH_MASK) << 32;
}

// ===========================================================================
// Two-touch super-tile kernel (16-byte aligned in/out).  One CTA per
// super-tile (dynamic id); warp w owns ROWS consecutive 512-byte rows:
//   phase 1  stream the slice from HBM (UNROLL rows in flight per warp,
//            L2 evict_last) and fold it; the block turns the slice folds into
//            slice offsets and the super-tile AGGREGATE, published at once;
//   phase 2  warp 0 looks back for the super-tile prefix; with EARLY the
//            other warps meanwhile load and locally scan their first UNROLL
//            rows of phase 3;
//   phase 3  every warp re-reads its slice (now L2-resident, evict_first),
//            scans it row by row and stores (STG.128, 512 B per warp).
// ===========================================================================
// P1U: rows in flight per warp in phase 1 (its only live state is the raw
// rows, so it can exceed phase 3's UNROLL).
template <int OP, typename T, typename Tin, int WARPS, int ROWS, int UNROLL, int DEPTH, bool NC, bool EXCLUSIVE,
          bool EARLY, int P1U = UNROLL, int PF_ROWS = 0, bool TRACE = false, int RB = 512>
__global__ void __launch_bounds__(WARPS * 32) scan_l2_kernel(ScanArgs<T, Tin> p, uint64_t *trace) {
  pdl_enter();
  using O = Op<OP, T>;
  // RB: input bytes per warp row — 512 (16 bytes per lane, LDG/STG.128) or
  // 1024 (32 bytes per lane, LDG/STG.256: half the memory instructions and
  // half the warp scans per element; used for the 8-byte and widened L shapes)
  static_assert(RB == 512 || RB == 1024, "row bytes");
  using Raw = std::conditional_t<RB == 1024, V32, uint4>;
  constexpr int E = RB / 32 / (int)sizeof(Tin);  // elements per lane per row
  constexpr int ROW = 32 * E;                     // elements per row
  constexpr bool LONG = ROWS * RB >= 16384;       // the L shape's 16 KiB slices (full / ragged bodies split)
  constexpr bool WIDEN = sizeof(T) != sizeof(Tin);
  static_assert(!WIDEN || (sizeof(T) == 8 && sizeof(Tin) == 4), "widening is 4 -> 8 bytes");
  constexpr int64_t TILE = (int64_t)WARPS * ROWS * ROW;
  static_assert(ROWS % UNROLL == 0 && ROWS % P1U == 0, "ROWS must be a multiple of UNROLL and P1U");
  static_assert(WARPS <= 32, "slice folds are scanned by one warp");
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ T s_slice[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T neutral = O::neutral();

  if (threadIdx.x == 0) {
    uint32_t t, e;
    draw_tile(p, t, e);
    s_tile = t;
    s_epoch = e;
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const uint32_t epoch = s_epoch;
  // TRACE (tools/lab/trace_l2.py only; compiled out otherwise): per tile
  // {start, phase 1 done, prefix known, stored, -, -, -, SM id} in ns
  auto stamp = [&](int k) {
    if constexpr (TRACE) {
      if (threadIdx.x == 0) trace[tile * 8 + k] = globaltimer_ns();
    }
  };
  if constexpr (TRACE) {
    if (threadIdx.x == 0) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      trace[tile * 8 + 7] = sm;
    }
  }
  stamp(0);
  const int64_t slice0 = tile * TILE + (int64_t)warp * ROWS * ROW;  // first element of my slice
  // The rest of the kernel is compiled twice (L shape): for full tiles (no
  // bounds checks at all) and for the one ragged last tile, where a lane goes
  // scalar only if its 16 bytes straddle n (before, the whole ragged tile
  // took scalar loads and stores and ran alone for ~16 us at the end of the
  // scan; profiles/r2_scan.md).
  const bool tile_full = tile * TILE + TILE <= p.n;
  auto tile_body = [&](auto full_tag) {
  constexpr bool full = decltype(full_tag)::value;  // false: the ragged tile (L), any tile (S, M)
  // a lane's 16 bytes at element i may use the vector path: always in a full
  // tile; in the L shape's ragged tile wherever they lie inside [0, n)
  auto vec_ok = [&](int64_t i) { return tile_full || (LONG && i + E <= p.n); };
  const uint64_t keep = l2::policy_evict_last();
  const uint64_t drop = l2::policy_evict_first();

  // A row stays in registers as its raw RB/32 input bytes per lane (4 or 8
  // registers for every T / Tin); it is unpacked and widened only where it is
  // folded, so the 8-byte and widened scans hold no more live state than
  // int32 at the same row width.
  auto ldv = [&](const Tin *a, uint64_t pol) -> Raw {
    if constexpr (RB == 1024) return l2::ldg256_hint<NC>(a, pol);
    else return l2::ldg128_hint<NC>(a, pol);
  };
  auto pack_in = [&](const Tin (&e)[E]) -> Raw {
    if constexpr (RB == 1024) {
      V32 w;
#pragma unroll
      for (int k = 0; k < E; ++k) vset<Tin>(w, k, e[k]);
      return w;
    } else {
      return Chunk<Tin>::pack(e);
    }
  };
  auto load_raw = [&](int r, uint64_t pol) -> Raw {
    const int64_t i = slice0 + (int64_t)r * ROW + lane * E;
    // the ragged last tile takes the vector path too wherever a lane's
    // bytes lie inside [0, n): only the lane straddling n goes scalar
    if constexpr (full) {
      return ldv(p.in + i, pol);
    } else {
      if (vec_ok(i)) return ldv(p.in + i, pol);
      Tin e[E];  // padding only reaches positions >= n (never stored)
#pragma unroll
      for (int k = 0; k < E; ++k) e[k] = i + k < p.n ? p.in[i + k] : Op<OP, Tin>::neutral();
      return pack_in(e);
    }
  };
  auto widen = [&](const Raw &raw, T (&v)[E]) {
    if constexpr (RB == 1024) {
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = (T)vget<Tin>(raw, k);
    } else {
      Tin e[E];
      Chunk<Tin>::unpack(raw, e);
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = (T)e[k];
    }
  };

  // phase 1: slice folds
  T acc = neutral;
#pragma unroll 1
  for (int r0 = 0; r0 < ROWS; r0 += P1U) {
    Raw raw[P1U];
#pragma unroll
    for (int u = 0; u < P1U; ++u) raw[u] = load_raw(r0 + u, keep);
#pragma unroll
    for (int u = 0; u < P1U; ++u) {
      T v[E];
      widen(raw[u], v);
#pragma unroll
      for (int k = 0; k < E; ++k) acc = O::fold(acc, v[k]);
    }
  }
  acc = warp_fold<OP, T>(acc);
  if (lane == 0) s_slice[warp] = acc;
  __syncthreads();
  stamp(1);

  // While warp 0 looks back (the SM has no HBM reads in flight then), every
  // warp asks the TMA unit to pull the first PF_ROWS rows of its slice of the
  // tile pf_dist ids ahead into L2 (cp.async.bulk.prefetch, evict_last): that
  // tile's phase 1 — a fraction of a wave later, on whichever SM draws it —
  // then runs on L2 hits, and the HBM reads move into this SM's idle time.
  // A hint only: results never depend on it.
  if constexpr (PF_ROWS > 0) {
    const int64_t nt = tile + p.pf_dist;
    if (p.pf_dist > 0 && lane == 0 && (nt + 1) * TILE <= p.n) {
      const Tin *a = p.in + nt * TILE + (int64_t)warp * ROWS * ROW;
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a),
                   "r"((uint32_t)(PF_ROWS * RB)), "l"(keep)
                   : "memory");
    }
  }

  // phase 2: slice offsets, aggregate, look-back (warp 0)
  if (warp == 0) {
    const T mine = lane < WARPS ? s_slice[lane] : neutral;
    const T w = warp_inclusive<OP, T>(mine, lane);
    const T wex = warp_exclusive_of<OP, T>(w, lane);
    const T total = __shfl_sync(0xffffffffu, w, WARPS - 1);
    T prefix;
    if (tile == 0) {
      prefix = lane == 0 ? carry_in<OP, T>(p) : neutral;
      prefix = __shfl_sync(0xffffffffu, prefix, 0);
      if (lane == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, O::fold(prefix, total));
    } else {
      if (lane == 0) p.status.publish(tile, epoch, FLAG_AGGREGATE, total);
      prefix = look_back<OP, T, DEPTH>(p.status, tile, epoch);
      if (lane == 0) p.status.publish(tile, epoch, FLAG_INCLUSIVE, O::fold(prefix, total));
    }
    if (lane < WARPS) s_slice[lane] = O::fold(prefix, wex);  // exclusive prefix of slice `lane`
    stamp(2);
  }

  // phase 3 helpers.  load_local: rows [r0, r0+UNROLL) into registers (raw),
  // each row's exclusive offset relative to the chunk start (off: the
  // warp-exclusive scan of the lanes' in-lane folds) and the chunk fold
  // (ctot).  store_chunk redoes the in-lane running fold v0 ⊕ .. ⊕ vk — the
  // same operations in the same order, so results do not change.
  auto load_local = [&](int r0, Raw (&raw)[UNROLL], T (&off)[UNROLL], T &ctot) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) raw[u] = load_raw(r0 + u, drop);
    ctot = neutral;
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      T v[E];
      widen(raw[u], v);
#pragma unroll
      for (int k = 1; k < E; ++k) v[k] = O::fold(v[k - 1], v[k]);
      const T x = warp_inclusive<OP, T>(v[E - 1], lane);
      off[u] = O::fold(ctot, warp_exclusive_of<OP, T>(x, lane));
      ctot = O::fold(ctot, __shfl_sync(0xffffffffu, x, 31));
    }
  };
  auto store_chunk = [&](int r0, const Raw (&raw)[UNROLL], const T (&off)[UNROLL], T base) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const T cb = O::fold(base, off[u]);
      T v[E], o[E];
      widen(raw[u], v);
#pragma unroll
      for (int k = 1; k < E; ++k) v[k] = O::fold(v[k - 1], v[k]);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if constexpr (EXCLUSIVE) o[k] = k == 0 ? cb : O::fold(cb, v[k - 1]);
        else o[k] = O::fold(cb, v[k]);
      }
      const int64_t i = slice0 + (int64_t)(r0 + u) * ROW + lane * E;
      bool vec = true;
      if constexpr (!full) vec = vec_ok(i);
      if (vec) {
        constexpr int OB = E * (int)sizeof(T);  // output bytes per lane: 16, 32 or 64
        if constexpr (OB == 16) {
          l2::stg128_hint(p.out + i, Chunk<T>::pack(o), drop);
        } else {
          constexpr int EPV = 32 / (int)sizeof(T);
#pragma unroll
          for (int h = 0; h < OB / 32; ++h) {
            V32 w;
#pragma unroll
            for (int k = 0; k < EPV; ++k) vset<T>(w, k, o[h * EPV + k]);
            l2::stg256v_hint(p.out + i + h * EPV, w, drop);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (i + k < p.n) p.out[i + k] = o[k];
      }
    }
  };
  Raw v0[UNROLL];
  T off0[UNROLL], ctot0;
  const bool early = EARLY && warp != 0;
  if (early) load_local(0, v0, off0, ctot0);
  __syncthreads();
  T base = s_slice[warp];
  if (!early) load_local(0, v0, off0, ctot0);
  store_chunk(0, v0, off0, base);
  base = O::fold(base, ctot0);
#pragma unroll 1
  for (int r0 = UNROLL; r0 < ROWS; r0 += UNROLL) {
    Raw v[UNROLL];
    T off[UNROLL], ctot;
    load_local(r0, v, off, ctot);
    store_chunk(r0, v, off, base);
    base = O::fold(base, ctot);
  }
  stamp(3);
  };
  // the split pays off for the long L-shape tiles; the short S/M ones keep one
  // (bounds-checked) body, which keeps them inside 64 registers
  if (LONG && tile_full) tile_body(std::integral_constant<bool, LONG>{});
  else tile_body(std::false_type{});
}

// ===========================================================================
// Register-tile fallback (arrays not 16-byte aligned): one tile of
// BLOCK x ITEMS consecutive elements per CTA, scalar loads/stores.
// ===========================================================================
template <int OP, typename T, typename Tin, int BLOCK, int ITEMS, int DEPTH, bool EXCLUSIVE>
__global__ void __launch_bounds__(BLOCK, 2) scan_reg_kernel(ScanArgs<T, Tin> p) {
  pdl_enter();
  using O = Op<OP, T>;
  constexpr int WARPS = BLOCK / 32;
  constexpr int64_t TILE = (int64_t)BLOCK * ITEMS;
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ T s_warp[WARPS];
  __shared__ T s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T neutral = O::neutral();

  if (threadIdx.x == 0) {
    uint32_t t, e;
    draw_tile(p, t, e);
    s_tile = t;
    s_epoch = e;
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const uint32_t epoch = s_epoch;
  const int64_t i0 = tile * TILE + (int64_t)threadIdx.x * ITEMS;

  T x[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) x[k] = (i0 + k < p.n) ? (T)p.in[i0 + k] : neutral;
#pragma unroll
  for (int k = 1; k < ITEMS; ++k) x[k] = O::fold(x[k - 1], x[k]);
  const T incl = warp_inclusive<OP, T>(x[ITEMS - 1], lane);
  const T excl_in_warp = warp_exclusive_of<OP, T>(incl, lane);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const T mine = lane < WARPS ? s_warp[lane] : neutral;
    const T w = warp_inclusive<OP, T>(mine, lane);
    const T wex = warp_exclusive_of<OP, T>(w, lane);
    const T total = __shfl_sync(0xffffffffu, w, WARPS - 1);
    T prefix;
    if (tile == 0) {
      prefix = lane == 0 ? carry_in<OP, T>(p) : neutral;
      prefix = __shfl_sync(0xffffffffu, prefix, 0);
      if (lane == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, O::fold(prefix, total));
    } else {
      if (lane == 0) p.status.publish(tile, epoch, FLAG_AGGREGATE, total);
      prefix = look_back<OP, T, DEPTH>(p.status, tile, epoch);
      if (lane == 0) p.status.publish(tile, epoch, FLAG_INCLUSIVE, O::fold(prefix, total));
    }
    if (lane < WARPS) s_warp[lane] = O::fold(prefix, wex);  // exclusive prefix of warp `lane`
  }
  __syncthreads();
  const T base = O::fold(s_warp[warp], excl_in_warp);  // exclusive prefix of my first element
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    T y;
    if constexpr (EXCLUSIVE) y = k == 0 ? base : O::fold(base, x[k - 1]);
    else y = O::fold(base, x[k]);
    if (i0 + k < p.n) p.out[i0 + k] = y;
  }
}

template <typename T>
size_t status_bytes(int64_t tiles) {
  return (size_t)tiles * 2 * sizeof(T);  // 8 (4-byte T) or 16 (8-byte T) tagged bytes per tile
}

// Fill the argument block for a tile size of tile_elems elements.
template <typename T, typename Tin = T>
ScanArgs<T, Tin> make_args(int64_t n, int64_t tile_elems, const void *in, void *out, const void *carry,
                           int64_t carry_count, void *ws) {
  ScanArgs<T, Tin> p;
  p.n = n;
  p.num_tiles = (n + tile_elems - 1) / tile_elems;
  p.in = static_cast<const Tin *>(in);
  p.out = static_cast<T *>(out);
  p.carry = static_cast<const T *>(carry);
  p.carry_count = carry_count;
  p.pf_dist = 0;
  char *w = static_cast<char *>(ws);
  p.ticket = reinterpret_cast<unsigned long long *>(w);
  p.status.word = reinterpret_cast<uint64_t *>(w + HEADER);  // same base for every T (see Status)
  return p;
}

}  // namespace scan_detail
}  // namespace ga
