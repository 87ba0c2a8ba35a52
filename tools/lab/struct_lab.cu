// struct_lab.cu — tuning lab only (round 2): streaming ceilings of the
// STRUCTURES a scan can take, with the look-back removed, so the cost of the
// structure and the cost of the look-back can be told apart.
//   v0..      twotouch: per CTA one super-tile of W warps x R rows x 512 B,
//             phase 1 streams it from HBM (evict_last), __syncthreads, phase 3
//             re-reads it (evict_first) and stores it.  ONE tile per CTA
//             (blockIdx.x) or PERSISTENT CTAs (grid = SMs, tiles strided),
//             optional L2 prefetch of the tile d ids ahead between phases.
//   v40..     smem single touch: per CTA a tile of TB bytes brought into
//             shared memory by cp.async.bulk (TMA, mbarrier) in 16 KiB
//             pieces, then stored by cp.async.bulk smem -> global.
//   v60..     plain 256-bit copy (the 1:1 ceiling).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld128(const void *p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st128(void *p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// ---------------------------------------------------------------- two-touch
template <int W, int R, int U, bool PERSIST, int PF>
__global__ void __launch_bounds__(W * 32) twotouch(const uint4 *in, uint4 *out, int64_t ntiles, int pfd,
                                                   uint32_t *sink) {
  constexpr int64_t TILE = (int64_t)W * R * 32;  // uint4 per tile
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t keep = pol_last(), drop = pol_first();
  for (int64_t t = blockIdx.x; t < ntiles; t += PERSIST ? gridDim.x : ntiles) {
    const int64_t s0 = t * TILE + (int64_t)warp * R * 32 + lane;
    uint32_t acc = 0;
#pragma unroll 1
    for (int r0 = 0; r0 < R; r0 += U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld128(in + s0 + (int64_t)(r0 + u) * 32, keep);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x9e3779b9u) *sink = acc;
    if constexpr (PF > 0) {
      const int64_t nt = t + pfd;
      if (lane == 0 && nt < ntiles)
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(
                         in + nt * TILE + (int64_t)warp * R * 32),
                     "r"((uint32_t)(R * 512)), "l"(keep)
                     : "memory");
    }
    __syncthreads();
#pragma unroll 1
    for (int r0 = 0; r0 < R; r0 += U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld128(in + s0 + (int64_t)(r0 + u) * 32, drop);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u].x += 1;
        st128(out + s0 + (int64_t)(r0 + u) * 32, v[u], drop);
      }
    }
  }
}

// ---------------------------------------------------------------- smem single touch (TMA bulk)
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int TB, int BLOCK, bool PERSIST>
__global__ void __launch_bounds__(BLOCK) smem_touch(const char *in, char *out, int64_t ntiles) {
  constexpr int PIECE = 16384;
  constexpr int NP = TB / PIECE;
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[NP];
  if (threadIdx.x == 0) {
    for (int i = 0; i < NP; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  const uint64_t drop = pol_first();
  for (int64_t t = blockIdx.x; t < ntiles; t += PERSIST ? gridDim.x : ntiles) {
    if (threadIdx.x == 0) {
      // the previous tile's bulk stores must have read smem before it is refilled
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      for (int i = 0; i < NP; ++i) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[i])), "r"(PIECE)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
            "%4;" ::"r"(sa(sm + i * PIECE)),
            "l"(in + t * TB + i * PIECE), "r"(PIECE), "r"(sa(&bar[i])), "l"(drop)
            : "memory");
      }
    }
    // every thread waits for every piece (stand-in for the fold over smem)
    uint32_t acc = 0;
    for (int i = 0; i < NP; ++i) {
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(sa(&bar[i])), "r"(phase)
            : "memory");
      acc += *reinterpret_cast<const uint32_t *>(sm + i * PIECE + threadIdx.x * 4);
    }
    phase ^= 1;
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int i = 0; i < NP; ++i)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                         out + t * TB + i * PIECE),
                     "r"(sa(sm + i * PIECE)), "r"(PIECE), "l"(drop)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (acc == 0x9e3779b9u) out[0] = 1;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---------------------------------------------------------------- 1:1 copy
template <int BLOCK, int UNROLL>
__global__ void __launch_bounds__(BLOCK) copy256(const uint4 *in, uint4 *out, int64_t nvec) {
  const int64_t base = (int64_t)blockIdx.x * BLOCK * UNROLL * 2 + threadIdx.x * 2;
  uint4 r[UNROLL][2];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + (int64_t)u * BLOCK * 2;
    if (i < nvec)
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[u][0].x), "=r"(r[u][0].y), "=r"(r[u][0].z), "=r"(r[u][0].w), "=r"(r[u][1].x),
                     "=r"(r[u][1].y), "=r"(r[u][1].z), "=r"(r[u][1].w)
                   : "l"(in + i));
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    const int64_t i = base + (int64_t)u * BLOCK * 2;
    if (i < nvec)
      asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + i),
                   "r"(r[u][0].x), "r"(r[u][0].y), "r"(r[u][0].z), "r"(r[u][0].w), "r"(r[u][1].x),
                   "r"(r[u][1].y), "r"(r[u][1].z), "r"(r[u][1].w)
                   : "memory");
  }
}

int sms() {
  static int n = 0;
  if (!n) {
    int d;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  }
  return n;
}

template <int W, int R, int U, bool PERSIST, int PF>
int tt(int64_t bytes, const void *in, void *out, uint32_t *sink, int pfd, int per_sm, cudaStream_t s) {
  constexpr int64_t TB = (int64_t)W * R * 512;
  const int64_t ntiles = bytes / TB;
  const int grid = PERSIST ? sms() * per_sm : (int)ntiles;
  twotouch<W, R, U, PERSIST, PF><<<grid, W * 32, 0, s>>>((const uint4 *)in, (uint4 *)out, ntiles, pfd, sink);
  return 0;
}

template <int TB, int BLOCK, bool PERSIST>
int st(int64_t bytes, const void *in, void *out, int per_sm, cudaStream_t s) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(smem_touch<TB, BLOCK, PERSIST>, cudaFuncAttributeMaxDynamicSharedMemorySize, TB);
    init = true;
  }
  const int64_t ntiles = bytes / TB;
  const int grid = PERSIST ? sms() * per_sm : (int)ntiles;
  smem_touch<TB, BLOCK, PERSIST><<<grid, BLOCK, TB, s>>>((const char *)in, (char *)out, ntiles);
  return 0;
}

}  // namespace

extern "C" int struct_lab(int v, int64_t bytes, const void *in, void *out, void *sink, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t *k = (uint32_t *)sink;
  switch (v) {
    // two-touch, one tile per CTA
    case 0: tt<24, 32, 8, false, 0>(bytes, in, out, k, 0, 1, s); break;
    case 1: tt<24, 32, 8, false, 32>(bytes, in, out, k, 42, 1, s); break;
    case 2: tt<24, 16, 8, false, 0>(bytes, in, out, k, 0, 1, s); break;
    case 3: tt<12, 32, 8, false, 0>(bytes, in, out, k, 0, 1, s); break;
    case 4: tt<32, 8, 8, false, 0>(bytes, in, out, k, 0, 1, s); break;
    case 5: tt<16, 16, 8, false, 0>(bytes, in, out, k, 0, 1, s); break;
    // two-touch, persistent
    case 10: tt<24, 32, 8, true, 0>(bytes, in, out, k, 0, 1, s); break;
    case 11: tt<24, 16, 8, true, 0>(bytes, in, out, k, 0, 1, s); break;
    case 12: tt<12, 32, 8, true, 0>(bytes, in, out, k, 0, 2, s); break;
    case 13: tt<16, 16, 8, true, 0>(bytes, in, out, k, 0, 2, s); break;
    // smem single touch (TMA bulk), one tile per CTA
    case 40: st<65536, 256, false>(bytes, in, out, 1, s); break;
    case 41: st<98304, 256, false>(bytes, in, out, 1, s); break;
    case 42: st<196608, 256, false>(bytes, in, out, 1, s); break;
    case 43: st<32768, 256, false>(bytes, in, out, 1, s); break;
    // smem single touch, persistent
    case 50: st<65536, 256, true>(bytes, in, out, 3, s); break;
    case 51: st<98304, 256, true>(bytes, in, out, 2, s); break;
    case 52: st<196608, 256, true>(bytes, in, out, 1, s); break;
    case 53: st<32768, 256, true>(bytes, in, out, 6, s); break;
    // 1:1 copy
    case 60: {
      const int64_t nvec = bytes / 16;
      copy256<256, 8><<<(int)((nvec + 4095) / 4096), 256, 0, s>>>((const uint4 *)in, (uint4 *)out, nvec);
      break;
    }
    default: return 2;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}
