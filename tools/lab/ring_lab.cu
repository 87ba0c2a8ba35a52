// ring_lab.cu — tuning lab only (round 2, third pass): a single-touch int32
// SUM scan whose tile waits for its prefix in REGISTERS, not in shared memory.
//
// Persistent CTAs (C per SM) draw tiles from a ticket.  Each CTA keeps a ring
// of S shared-memory stages filled by TMA bulk loads; a tile is copied from
// its stage into registers (R rows of 512 B per warp, 16 B per lane per row)
// and the stage is refilled with the CTA's next tile at once, so the load of
// tile k+S overlaps the fold, look-back, scan and store of tile k.  The
// look-back walks 256 statuses per round trip and stops at the nearest
// INCLUSIVE, or at the CTA's own previous tile (whose inclusive value it
// kept).  Status word = {epoch:30 | flag:2 | 32 value bits}.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

constexpr uint32_t F_AGG = 1, F_INC = 2;

__device__ __forceinline__ uint64_t tagw(uint32_t epoch, uint32_t flag, int32_t v) {
  return ((uint64_t)((epoch << 2) | flag) << 32) | (uint32_t)v;
}

__device__ __forceinline__ void mb_wait(const uint64_t *b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(sa(b)), "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mb_init(uint64_t *b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count));
}

// Warp roles: 0..W-1 data (copy the tile into registers as soon as it lands,
// release the stage, wait for the prefix, scan, store); W producer (tickets,
// bulk loads); W+1 look-back; W+2..W+1+F fold (fold each stage from shared
// memory as it lands and publish its AGGREGATE at once, so no CTA's
// aggregate waits for its own earlier look-backs).
template <int W, int R, int S, int F, int C, bool EX, int PIECES>
__global__ void __launch_bounds__((W + 2 + F) * 32, C)
    ring_scan(const int32_t *__restrict__ in, int32_t *__restrict__ out, int64_t ntiles, uint64_t *status,
              unsigned long long *ticket, uint32_t epoch) {
  constexpr int TB = W * R * 512;  // tile bytes
  constexpr int TE = TB / 4;       // tile elements
  constexpr int PB = TB / PIECES;  // bytes per bulk copy
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[S], empty[S], folded[S], pref[S];
  __shared__ int64_t tile_of[S];
  __shared__ int32_t aggsm[S], presm[S];
  __shared__ int32_t wt[2][W];
  __shared__ int32_t ft[F];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], W + F);
      mb_init(&folded[s], 1);
      mb_init(&pref[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (w == W) {  // ---------------------------------------------------------- producer
    if (lane != 0) return;
    const uint64_t drop = pol_first();
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      if (k >= S) mb_wait(&empty[s], (uint32_t)((k / S - 1) & 1));
      const int64_t t = (int64_t)atomicAdd(ticket, 1ull);
      tile_of[s] = t;
      if (t >= ntiles) {
        mb_arrive(&full[s]);  // sentinel: wakes the consumers, who stop
        return;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(TB) : "memory");
      const char *src = reinterpret_cast<const char *>(in) + t * (int64_t)TB;
#pragma unroll
      for (int i = 0; i < PIECES; ++i)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
            "[%3], %4;" ::"r"(sa(smem + s * TB + i * PB)),
            "l"(src + i * PB), "r"(PB), "r"(sa(&full[s])), "l"(drop)
            : "memory");
    }
  }

  if (w >= W + 2) {  // ------------------------------------------------------ fold
    const int f = w - (W + 2);
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      mb_wait(&full[s], (uint32_t)((k / S) & 1));
      const int64_t t = *reinterpret_cast<volatile int64_t *>(&tile_of[s]);
      if (t >= ntiles) return;
      int32_t a = 0;
      const char *p = smem + s * TB + (f * 32 + lane) * 16;
#pragma unroll 8
      for (int i = 0; i < TB / (F * 512); ++i) {
        const int4 q = *reinterpret_cast<const int4 *>(p + i * F * 512);
        a += q.x + q.y + q.z + q.w;
      }
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
#pragma unroll
      for (int d = 16; d; d >>= 1) a += __shfl_xor_sync(0xffffffffu, a, d);
      if (F > 1) {
        if (lane == 0) ft[f] = a;
        asm volatile("bar.sync 2, %0;" ::"n"(F * 32) : "memory");
        if (f == 0) {
          a = 0;
          for (int i = 0; i < F; ++i) a += ft[i];
        }
        asm volatile("bar.sync 2, %0;" ::"n"(F * 32) : "memory");
      }
      if (f == 0 && lane == 0) {
        st_relaxed(status + t, tagw(epoch, t == 0 ? F_INC : F_AGG, a));
        aggsm[s] = a;
        mb_arrive(&folded[s]);
      }
    }
  }

  if (w == W + 1) {  // ------------------------------------------------------ look-back
    int64_t prev_t = -1;  // this CTA's previous tile and its inclusive value
    int32_t prev_inc = 0;
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      mb_wait(&full[s], (uint32_t)((k / S) & 1));
      const int64_t t = *reinterpret_cast<volatile int64_t *>(&tile_of[s]);
      if (t >= ntiles) return;
      mb_wait(&folded[s], (uint32_t)((k / S) & 1));
      const int32_t agg = *reinterpret_cast<volatile int32_t *>(&aggsm[s]);
      int32_t P = 0;
      if (t > 0) {
        int64_t base = t - 1;
        for (;;) {
          uint64_t sw[8];
          int dstop;
          for (;;) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int64_t idx = base - (j * 32 + lane);
              sw[j] = (idx >= 0 && idx != prev_t) ? ld_relaxed(status + idx) : 0;
            }
            dstop = 256;
            bool ok = true;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int64_t idx = base - (j * 32 + lane);
              const uint32_t hi = (uint32_t)(sw[j] >> 32);
              const bool stop = idx < 0 || idx == prev_t || hi == ((epoch << 2) | F_INC);
              const unsigned m = __ballot_sync(0xffffffffu, stop);
              if (m && dstop == 256) dstop = j * 32 + __ffs(m) - 1;
              if (j * 32 + lane <= dstop && !stop && hi != ((epoch << 2) | F_AGG)) ok = false;
            }
            if (__all_sync(0xffffffffu, ok)) break;
          }
          int32_t part = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int64_t idx = base - (j * 32 + lane);
            if (j * 32 + lane <= dstop && idx >= 0) part += idx == prev_t ? prev_inc : (int32_t)(uint32_t)sw[j];
          }
#pragma unroll
          for (int d = 16; d; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
          P += part;
          if (dstop < 256) break;
          base -= 256;
        }
        if (lane == 0) st_relaxed(status + t, tagw(epoch, F_INC, P + agg));
      }
      prev_t = t;
      prev_inc = P + agg;
      if (lane == 0) {
        presm[s] = P;
        mb_arrive(&pref[s]);
      }
      __syncwarp();
    }
  }

  if (w < W) {  // ------------------------------------------------------------ data
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      const uint32_t ph = (uint32_t)((k / S) & 1);
      mb_wait(&full[s], ph);
      const int64_t t = *reinterpret_cast<volatile int64_t *>(&tile_of[s]);
      if (t >= ntiles) return;
      uint4 v[R];
      const char *st = smem + s * TB + (w * R) * 512 + lane * 16;
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = *reinterpret_cast<const uint4 *>(st + r * 512);
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
      int32_t a = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) a += (int32_t)v[r].x + (int32_t)v[r].y + (int32_t)v[r].z + (int32_t)v[r].w;
#pragma unroll
      for (int d = 16; d; d >>= 1) a += __shfl_xor_sync(0xffffffffu, a, d);
      if (lane == 0) wt[k & 1][w] = a;
      asm volatile("bar.sync 3, %0;" ::"n"(W * 32) : "memory");
      int32_t carry = 0;
      for (int i = 0; i < w; ++i) carry += wt[k & 1][i];
      mb_wait(&pref[s], ph);
      carry += *reinterpret_cast<volatile int32_t *>(&presm[s]);
      int32_t *dst = out + t * (int64_t)TE + (w * R) * 128 + lane * 4;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int32_t s0 = (int32_t)v[r].x, s1 = s0 + (int32_t)v[r].y, s2 = s1 + (int32_t)v[r].z,
                      s3 = s2 + (int32_t)v[r].w;
        int32_t x = s3;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x += y;
        }
        const int32_t b = carry + x - s3;
        carry += __shfl_sync(0xffffffffu, x, 31);
        int4 o;
        if (EX) {
          o.x = b;
          o.y = b + s0;
          o.z = b + s1;
          o.w = b + s2;
        } else {
          o.x = b + s0;
          o.y = b + s1;
          o.z = b + s2;
          o.w = b + s3;
        }
        asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(dst + r * 128), "r"(o.x),
                     "r"(o.y), "r"(o.z), "r"(o.w)
                     : "memory");
      }
    }
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

template <int W, int R, int S, int F, int C, int PIECES>
int run(int ex, int64_t n, const int32_t *in, int32_t *out, uint64_t *status, unsigned long long *ticket,
        uint32_t epoch, cudaStream_t st) {
  constexpr int TB = W * R * 512;
  constexpr int TE = TB / 4;
  if (n % TE) return 3;
  const int64_t ntiles = n / TE;
  auto k0 = ring_scan<W, R, S, F, C, false, PIECES>;
  auto k1 = ring_scan<W, R, S, F, C, true, PIECES>;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, S * TB);
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, S * TB);
    init = true;
  }
  int grid = sms() * C;
  if (grid > ntiles) grid = (int)ntiles;
  (ex ? k1 : k0)<<<grid, (W + 2 + F) * 32, S * TB, st>>>(in, out, ntiles, status, ticket, epoch);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

}  // namespace

// id: W warps, R rows per warp (512 B), S stages, C CTAs per SM
// id: W data warps, R rows per warp (512 B), S stages, F fold warps, C CTAs per SM, bulk pieces
#define V(X)                \
  X(0, 16, 8, 3, 2, 1, 4)   \
  X(1, 16, 4, 6, 2, 1, 2)   \
  X(2, 8, 8, 3, 1, 2, 2)    \
  X(3, 16, 8, 3, 4, 1, 4)   \
  X(4, 8, 16, 3, 2, 1, 4)   \
  X(5, 16, 4, 3, 2, 2, 2)   \
  X(6, 16, 16, 1, 2, 1, 8)  \
  X(7, 8, 8, 2, 1, 3, 2)    \
  X(8, 16, 8, 2, 2, 1, 4)   \
  X(9, 16, 4, 4, 2, 1, 2)

extern "C" int ring_lab(int v, int ex, int64_t n, const void *in, void *out, void *status, void *ticket,
                        uint32_t epoch, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t *i = (const int32_t *)in;
  int32_t *o = (int32_t *)out;
  uint64_t *stt = (uint64_t *)status;
  unsigned long long *tk = (unsigned long long *)ticket;
  switch (v) {
#define C(id, W, R, S, F, CC, P) \
  case id: return run<W, R, S, F, CC, P>(ex, n, i, o, stt, tk, epoch, s);
    V(C)
#undef C
  }
  return 2;
}
extern "C" int ring_lab_tile_elems(int v) {
  switch (v) {
#define C(id, W, R, S, F, CC, P) \
  case id: return W * R * 128;
    V(C)
#undef C
  }
  return 0;
}
