// reduce_kernel.cuh — the single-pass map-reduce kernel (see reduce.cu for
// the algorithm and its citations), templated on its CTA shape so reduce.cu
// instantiates the tuned one and tools/lab can time others.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string.h>

#include <algorithm>
#include <type_traits>

#include "ga_device.cuh"
#include "ga_host.h"

namespace ga {
namespace red_detail {


constexpr int RED_MAX_PARTIALS = 32768;
constexpr int RED_GROUP = 128;  // blocks per first-level group of the finish (at least)
constexpr int RED_MAX_GROUPS = 256;
// Workspace layout (zeroed once by the caller): the call epoch (u32) in its
// own 128-byte line, then one 32-byte slot per block partial, then one per
// group partial.  A slot holds the value (<= 16 bytes) and the tag of the
// call that wrote it (see grid_finish).
constexpr size_t RED_HEADER = 128;
constexpr size_t RED_SLOT = 32;  // the largest slot (16-byte values); see slot_stride
constexpr size_t RED_GSLOT_OFF = RED_HEADER + (size_t)RED_MAX_PARTIALS * RED_SLOT;
constexpr size_t RED_WS_BYTES = RED_GSLOT_OFF + (size_t)RED_MAX_GROUPS * RED_SLOT;
constexpr uint32_t RED_EPOCH_MASK = 0x7fffffffu;

// What a kernel needs to finish: the workspace and the group size (host:
// finish_group()).
struct Finish {
  char *ws;
  int group;
};

// Host: the finish of a `grid`-block launch of a kernel with at least
// `minb` co-resident blocks per SM.  Groups of RED_GROUP blocks (more when
// the grid would need over RED_MAX_GROUPS groups), and fewer groups than
// co-resident blocks so that the waiting group leaders can never starve the
// blocks they wait for (every full B200 launch: 128).
inline Finish make_finish(void *ws, int64_t grid, int minb) {
  const int64_t resident = (int64_t)sm_count() * minb;
  const int64_t max_groups = std::max<int64_t>(1, std::min<int64_t>(RED_MAX_GROUPS, resident - 1));
  Finish f;
  f.ws = static_cast<char *>(ws);
  f.group = (int)std::max<int64_t>(RED_GROUP, (grid + max_groups - 1) / max_groups);
  return f;
}

template <typename T>
__host__ __device__ constexpr bool is_fp() {
  return std::is_floating_point<T>::value;
}

// Map (over index i) then accumulate into the reduction's accumulator.
// SUM over floats accumulates in Tacc with one fused multiply-add per term
// (exact product, one rounding): the tolerance of DESIGN.md R9/R10 applies.
// SUM over integers widens to Tacc, then wraps (R3, R4).  MAX/MIN evaluate
// the map in Tin with RN / wrap (R3) and fold with maxNum/minNum (R6).
// Complex SUM (NEXT-3): x | x*y | conj(x)*y accumulated with FMAs per
// component (tolerance-governed, like real float SUM); x*x under SQUARE means
// |x|^2 into a real accumulator.
template <typename Tin, typename Tacc, int MAP>
__device__ __forceinline__ Tacc map_acc_complex(Tacc acc, Tin x, Tin y) {
  if constexpr (!is_complex<Tacc>::value) {  // |x|^2
    return e_fma(x.im, x.im, e_fma(x.re, x.re, acc));
  } else if constexpr (MAP == GA_MAP_ID) {
    return e_add(acc, x);
  } else {
    const decltype(x.re) s = MAP == GA_MAP_CONJ_MUL ? -1 : 1;  // conj flips the sign of x.im
    Tacc r;
    r.re = e_fma(-s * x.im, y.im, e_fma(x.re, y.re, acc.re));
    r.im = e_fma(s * x.im, y.re, e_fma(x.re, y.im, acc.im));
    return r;
  }
}

template <typename Tin, typename Tacc, int OP, int MAP>
__device__ __forceinline__ Tacc map_acc(Tacc acc, Tin x, Tin y) {
  if constexpr (is_complex<Tin>::value) {
    return map_acc_complex<Tin, Tacc, MAP>(acc, x, y);
  } else if constexpr (OP == GA_OP_SUM) {
    const Tacc u = (Tacc)x;
    if constexpr (is_fp<Tacc>()) {
      if constexpr (MAP == GA_MAP_ID) return e_add(acc, u);
      else if constexpr (MAP == GA_MAP_MUL) return e_fma(u, (Tacc)y, acc);
      else return e_fma(u, u, acc);
    } else {
      if constexpr (MAP == GA_MAP_ID) return e_add(acc, u);
      else if constexpr (MAP == GA_MAP_MUL) return e_add(acc, e_mul(u, (Tacc)y));
      else return e_add(acc, e_mul(u, u));
    }
  } else {
    Tin t;
    if constexpr (MAP == GA_MAP_ID) t = x;
    else if constexpr (MAP == GA_MAP_MUL) t = e_mul(x, y);
    else t = e_mul(x, x);
    return Op<OP, Tacc>::fold(acc, (Tacc)t);
  }
}

template <typename Tin, typename Tacc>
struct RedArgs {
  int64_t n;
  int64_t head;  // elements folded by the scalar loop before the aligned body
  int64_t nvec;  // 32-byte vectors in the body
  const Tin *x;
  const Tin *y;
  Tacc *out;
  Finish fin;
  Exchange xg;  // cross-GPU finish (world == 0: none)
};

__device__ __forceinline__ void st_release_sys_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Cross-GPU finish (thread 0 of the last block), §8(f) NEXT-1: publish the
// local result into slot `rank` of every rank's exchange buffer (peer
// pointers: NVLink-mapped symmetric memory), then wait for all `world` slots
// of the own buffer and fold them in rank order, so every rank computes the
// same bits with no separate collective launch (prefix_only: the fold of the
// ranks before this one — the offset of a sharded scan).  Slot entry (32 B) =
// {value: 16 B, seq: 8 B, pad}; slots are double-buffered by seq parity (a
// rank cannot publish call seq+2 before every rank has read call seq).
template <int OP, typename Tacc>
__device__ Tacc exchange_fold(const Exchange &xg, Tacc local) {
  const int par = (int)(xg.seq & 1);
  for (int r = 0; r < xg.world; ++r) {
    char *e = reinterpret_cast<char *>(xg.peers[r]) + ((size_t)par * XG_MAX_WORLD + xg.rank) * XG_SLOT;
    *reinterpret_cast<Tacc *>(e) = local;
    st_release_sys_u64(reinterpret_cast<unsigned long long *>(e + 16), xg.seq);
  }
  const char *own = reinterpret_cast<const char *>(xg.peers[xg.rank]);
  Tacc v = Op<OP, Tacc>::neutral();
  for (int r = 0; r < xg.world; ++r) {
    const char *e = own + ((size_t)par * XG_MAX_WORLD + r) * XG_SLOT;
    const unsigned long long *f = reinterpret_cast<const unsigned long long *>(e + 16);
    uint32_t spins = 0;
    uint64_t t0 = 0;
    while (ld_acquire_sys_u64(f) != xg.seq) {
      if ((++spins & 1023u) == 0) {
        uint64_t now;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > 10000000000ull) __trap();  // a rank never arrived
      }
    }
    // every rank is waited for (slot-reuse safety); prefix_only folds r < rank
    if (!xg.prefix_only || r < xg.rank) v = Op<OP, Tacc>::fold(v, ldcg<Tacc>(reinterpret_cast<const Tacc *>(e)));
  }
  return v;
}

// Block-wide fold; result valid in thread 0.  Fixed order.
template <int OP, int BLOCK, typename T>
__device__ __forceinline__ T block_fold(T v, T *smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_fold<OP, T>(v);
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < BLOCK / 32 ? smem[lane] : Op<OP, T>::neutral();
    v = warp_fold<OP, T>(v);
  }
  return v;
}

// Tagged partial slots.  The tag of a call is its epoch + 1 (never 0, so a
// zeroed workspace holds no valid slot).  A value of S bytes is stored as
// S/4 64-bit words {tag:32 | 32 value bits}, each written with one relaxed
// 64-bit store (single-copy atomic) and read with relaxed loads: a reader that
// sees the call's tag in every word holds that call's value — no fence, no
// atomic, no release/acquire pair on either side.
__device__ __forceinline__ uint32_t finish_tag(const Finish &f) {
  uint32_t e;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(e) : "l"(f.ws) : "memory");
  return (e & RED_EPOCH_MASK) + 1u;
}

// Slots are packed at their own size (2 x sizeof(Tacc): one 8-byte word per
// 4 value bytes), so consecutive blocks fill whole 32-byte sectors.
template <typename Tacc>
__host__ __device__ constexpr size_t slot_stride() {
  return 2 * sizeof(Tacc);
}

template <typename Tacc>
__device__ __forceinline__ void slot_publish(char *slot, uint32_t tag, Tacc v) {
  constexpr int W = sizeof(Tacc) / 4;
  static_assert(W * 4 == sizeof(Tacc) && W * 8 <= RED_SLOT, "slot holds up to 16-byte values");
  uint32_t bits[W];
  memcpy(bits, &v, sizeof(Tacc));
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const uint64_t w = ((uint64_t)tag << 32) | bits[k];
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(slot + 8 * k), "l"(w) : "memory");
  }
}

// Spin (with a short sleep between polls) until every word of the slot
// carries `tag`, then return the value.  A slot that never arrives (a block
// that cannot run) traps after 10 s instead of hanging.
template <typename Tacc>
__device__ __forceinline__ Tacc slot_wait(const char *slot, uint32_t tag) {
  constexpr int W = sizeof(Tacc) / 4;
  uint32_t bits[W];
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (true) {
    bool ready = true;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      uint64_t w;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(slot + 8 * k) : "memory");
      ready = ready && (uint32_t)(w >> 32) == tag;
      bits[k] = (uint32_t)w;
    }
    if (ready) break;
    __nanosleep(64);
    if ((++spins & 1023u) == 0) {
      uint64_t now;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > 10000000000ull) __trap();
    }
  }
  Tacc v;
  memcpy(&v, bits, sizeof(Tacc));
  return v;
}

// Fold slots [0, count) of `base` in a fixed order — thread t folds t,
// t + BLOCK, ... then the block tree — with slot count-1 replaced by `own`
// (the caller's value, which it never published).  Result valid in thread 0.
template <int OP, int BLOCK, typename Tacc>
__device__ __forceinline__ Tacc fold_slots(const char *base, int count, uint32_t tag, Tacc own, Tacc *smem) {
  Tacc w = Op<OP, Tacc>::neutral();
  for (int i = threadIdx.x; i < count; i += BLOCK)
    w = Op<OP, Tacc>::fold(w, i == count - 1 ? own : slot_wait<Tacc>(base + (size_t)i * slot_stride<Tacc>(), tag));
  __syncthreads();  // smem reuse
  return block_fold<OP, BLOCK, Tacc>(w, smem);
}

// Grid finish (§8(a) a4), called by every thread of every block with the
// block's partial v (valid in thread 0) and the call's tag (finish_tag,
// loaded at kernel start).  Blocks form groups of f.group consecutive ids.
// A block that is not the last of its group publishes its partial into its
// tagged slot and exits — no fence, no atomic, no wait.  The LAST block of a
// group waits for the group's slots and folds them in index order (its own
// partial last); the last block of the grid then waits for the group
// partials, folds them in group order, runs the cross-GPU exchange if any,
// writes *out and advances the epoch (stream order makes it visible to the
// next call).  With one group the second level is skipped.  Only group
// leaders wait, and only for blocks that never wait, so progress needs more
// co-resident blocks than groups (make_finish() guarantees it; a starved
// wait traps after 10 s).  Every fold order depends on (grid, group) only.
template <int OP, int BLOCK, typename Tacc>
__device__ __forceinline__ void grid_finish(Tacc v, uint32_t tag, Tacc *smem, const Finish &f, Tacc *out,
                                            const Exchange &xg) {
  __shared__ Tacc s_own;
  const int grid = (int)gridDim.x, b = (int)blockIdx.x;
  const int ngroups = (grid + f.group - 1) / f.group;
  const int g = b / f.group;
  const int gsize = min(f.group, grid - g * f.group);
  char *slots = f.ws + RED_HEADER;
  char *gslots = f.ws + RED_GSLOT_OFF;
  if (b != g * f.group + gsize - 1) {
    if (threadIdx.x == 0) slot_publish<Tacc>(slots + (size_t)b * slot_stride<Tacc>(), tag, v);
    return;
  }
  if (threadIdx.x == 0) s_own = v;
  __syncthreads();
  Tacc w = fold_slots<OP, BLOCK, Tacc>(slots + (size_t)g * f.group * slot_stride<Tacc>(), gsize, tag, s_own, smem);
  if (ngroups > 1) {
    if (b != grid - 1) {
      if (threadIdx.x == 0) slot_publish<Tacc>(gslots + (size_t)g * slot_stride<Tacc>(), tag, w);
      return;
    }
    __syncthreads();  // every thread has read s_own
    if (threadIdx.x == 0) s_own = w;
    __syncthreads();
    w = fold_slots<OP, BLOCK, Tacc>(gslots, ngroups, tag, s_own, smem);
  }
  if (threadIdx.x == 0) {
    if (xg.world > 0) w = exchange_fold<OP, Tacc>(xg, w);
    *out = w;
    *reinterpret_cast<volatile uint32_t *>(f.ws) = tag & RED_EPOCH_MASK;  // the next call's epoch
  }
}

template <typename Tin, typename Tacc, int OP, int MAP, int UNROLL, int RED_BLOCK, int MINB>
__global__ void __launch_bounds__(RED_BLOCK, MINB) reduce_kernel(RedArgs<Tin, Tacc> p) {
  pdl_enter();
  constexpr int VEC = 32 / sizeof(Tin);
  constexpr bool HAS_Y = MAP == GA_MAP_MUL || MAP == GA_MAP_CONJ_MUL;
  __shared__ Tacc smem[RED_BLOCK / 32];

  const uint32_t tag = finish_tag(p.fin);
  const int64_t tid = (int64_t)blockIdx.x * RED_BLOCK + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * RED_BLOCK;

  Tacc acc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) acc[k] = Op<OP, Tacc>::neutral();

  // Scalar parts: the unaligned head (all of x when x/y are not co-aligned)
  // and the tail after the last whole vector.
  for (int64_t i = tid; i < p.head; i += nthreads)
    acc[0] = map_acc<Tin, Tacc, OP, MAP>(acc[0], p.x[i], HAS_Y ? p.y[i] : zero_of<Tin>());
  const int64_t tail0 = p.head + p.nvec * VEC;
  for (int64_t i = tail0 + tid; i < p.n; i += nthreads)
    acc[VEC - 1] = map_acc<Tin, Tacc, OP, MAP>(acc[VEC - 1], p.x[i], HAS_Y ? p.y[i] : zero_of<Tin>());

  const char *xb = reinterpret_cast<const char *>(p.x + p.head);
  const char *yb = HAS_Y ? reinterpret_cast<const char *>(p.y + p.head) : nullptr;
  constexpr int64_t CHUNK = (int64_t)RED_BLOCK * UNROLL;
  // Out-of-range vectors are filled with an input whose mapped value is the
  // neutral element (0 for SUM under any map; the neutral itself for MAX/MIN
  // under the identity map), so the accumulation is unconditional.  MAX/MIN
  // under x*y or x*x have no such input and keep the guard.
  constexpr bool FILL = OP == GA_OP_SUM || MAP == GA_MAP_ID;
  V32 fill;
#pragma unroll
  for (int k = 0; k < VEC; ++k) {
    if constexpr (OP == GA_OP_SUM) vset<Tin>(fill, k, zero_of<Tin>());
    else vset<Tin>(fill, k, (Tin)Op<OP, Tacc>::neutral());
  }
  // One batch: UNROLL vectors per input, RED_BLOCK apart, all loaded before
  // any is used; out-of-range vectors take the neutral fill.
  auto batch = [&](int64_t base) {
    V32 vx[UNROLL], vy[UNROLL];
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      const int64_t v = base + j * RED_BLOCK;
      if (v < p.nvec) {
        vx[j] = ld_nc_256(xb + v * 32);
        if constexpr (HAS_Y) vy[j] = ld_nc_256(yb + v * 32);
      } else {
        vx[j] = fill;
        vy[j] = fill;
      }
    }
#pragma unroll
    for (int j = 0; j < UNROLL; ++j)
      if (FILL || base + j * RED_BLOCK < p.nvec) {
#pragma unroll
        for (int k = 0; k < VEC; ++k)
          acc[k] = map_acc<Tin, Tacc, OP, MAP>(acc[k], vget<Tin>(vx[j], k), HAS_Y ? vget<Tin>(vy[j], k) : zero_of<Tin>());
      }
  };
  // The first batch is peeled out of the loop (the loop only runs when the
  // grid was capped): ptxas then schedules it like straight-line code — all
  // loads first — instead of squeezing the loop body into 32 registers.
  const int64_t base0 = (int64_t)blockIdx.x * CHUNK + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * CHUNK;
  if (base0 < p.nvec) batch(base0);
#pragma unroll 1
  for (int64_t base = base0 + stride; base < p.nvec; base += stride) batch(base);

  // Lane tree: ((a0+a4)+(a2+a6)) + ((a1+a5)+(a3+a7)) for VEC = 8.
#pragma unroll
  for (int w = VEC / 2; w >= 1; w >>= 1) {
#pragma unroll
    for (int k = 0; k < w; ++k) acc[k] = Op<OP, Tacc>::fold(acc[k], acc[k + w]);
  }
  Tacc v = block_fold<OP, RED_BLOCK, Tacc>(acc[0], smem);

  grid_finish<OP, RED_BLOCK, Tacc>(v, tag, smem, p.fin, p.out, p.xg);
}

template <typename Tacc, int OP>
__global__ void neutral_kernel(Tacc *out) {
  pdl_enter();
  *out = Op<OP, Tacc>::neutral();
}

}  // namespace red_detail
}  // namespace ga
