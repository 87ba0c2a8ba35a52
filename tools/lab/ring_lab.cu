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

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace slots per tile: 0 issue, 1 landed (fold start), 2 aggregate published, 3 look-back start,
// 4 prefix known, 5 data: stage copied to registers, 6 data: prefix seen, 7 data: stored (+smid in 7's high bits no)
#define TRC(slot) \
  if (trace) trace[(t) * 8 + (slot)] = gtime();

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
// bulk loads); W+1..W+NLB look-back (warp j takes uses j, j+NLB, ...);
// the last F fold (fold each stage from shared memory as it lands and
// publish its AGGREGATE at once, so no CTA's aggregate waits for its own
// earlier look-backs).  Per-use values live in rings of TR slots (tile id,
// aggregate, prefix + their mbarriers), so a role that runs ahead of another
// never overwrites what the slower one still needs.
template <int W, int R, int S, int F, int NLB, int C, bool EX, int PIECES, int LBM, bool DB>
__global__ void __launch_bounds__((W + 1 + NLB + F) * 32, C)
    ring_scan(const int32_t *__restrict__ in, int32_t *__restrict__ out, int64_t ntiles, uint64_t *status,
              unsigned long long *ticket, uint32_t epoch, uint64_t *trace) {
  constexpr int TB = W * R * 512;  // tile bytes
  constexpr int TE = TB / 4;       // tile elements
  constexpr int PB = TB / PIECES;  // bytes per bulk copy
  constexpr int TR = 16;
  static_assert(TR >= S + NLB + 2, "ring too short");
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[S], empty[S], folded[TR], pref[TR];
  __shared__ int64_t tid_ring[TR];
  __shared__ int64_t issued;
  __shared__ int32_t agg_ring[TR], pre_ring[TR];
  __shared__ int32_t wt[3][W];
  __shared__ int32_t ft[F];
  __shared__ int32_t incl_sm[LBM == 2 ? 512 : 1];
  constexpr bool EARLY = LBM == 1;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], W + F);
    }
    for (int i = 0; i < TR; ++i) {
      mb_init(&folded[i], 1);
      mb_init(&pref[i], 1);
    }
    issued = 0;
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
      tid_ring[k % TR] = t;
      if (t >= ntiles) {
        // sentinel for the data and fold warps (this use) and for every
        // look-back warp (the next NLB uses)
        for (int i = 1; i <= NLB; ++i) tid_ring[(k + i) % TR] = t;
        __threadfence_block();
        *reinterpret_cast<volatile int64_t *>(&issued) = k + 1 + NLB;
        mb_arrive(&full[s]);
        return;
      }
      __threadfence_block();
      *reinterpret_cast<volatile int64_t *>(&issued) = k + 1;
      TRC(0)
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

  if (w > W + NLB) {  // ------------------------------------------------------ fold
    const int f = w - (W + 1 + NLB);
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      mb_wait(&full[s], (uint32_t)((k / S) & 1));
      const int64_t t = *reinterpret_cast<volatile int64_t *>(&tid_ring[k % TR]);
      if (t >= ntiles) return;
      if (f == 0 && lane == 0) TRC(1)
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
        agg_ring[k % TR] = a;
        mb_arrive(&folded[k % TR]);
        TRC(2)
      }
    }
  }

  if (LBM == 2 && w == W + 1) {  // ---------------------------------- frontier look-back
    // base = the last position whose inclusive value is known (-1: none, 0);
    // each round reads the statuses after it up to the CTA's latest issued
    // tile (one round trip, <= 512 statuses), takes the longest ready run,
    // computes the inclusive values along it (INCLUSIVE statuses reset the
    // running value), hands every own tile inside it its prefix and moves
    // base to the end of the run.  No tile waits for another tile's
    // look-back: only for its predecessors' aggregates.
    int64_t base = -1;
    int32_t base_inc = 0;
    int64_t kr = 0;  // next own use to resolve
    for (;;) {
      int64_t kk = *reinterpret_cast<volatile int64_t *>(&issued);
      kk = __shfl_sync(0xffffffffu, kk, 0);  // one snapshot for the whole warp
      if (kk <= kr) {
        __nanosleep(64);
        continue;
      }
      const int64_t t0 = *reinterpret_cast<volatile int64_t *>(&tid_ring[kr % TR]);
      if (t0 >= ntiles) return;
      int64_t thi = *reinterpret_cast<volatile int64_t *>(&tid_ring[(kk - 1) % TR]);
      if (thi >= ntiles) thi = ntiles;
      int64_t wend = thi - 1;  // last position needed
      if (wend > base + 512) wend = base + 512;
      uint64_t sw[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t pos = base + 1 + j * 32 + lane;
        sw[j] = pos <= wend ? ld_relaxed(status + pos) : 0;
      }
      // the ready run [base+1, f-1]
      int64_t f = wend + 1;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t hi = (uint32_t)(sw[j] >> 32);
        const bool rdy = hi == ((epoch << 2) | F_INC) || hi == ((epoch << 2) | F_AGG);
        const int64_t pos = base + 1 + j * 32 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, !rdy && pos <= wend);
        if (m && f == wend + 1) f = base + 1 + j * 32 + __ffs(m) - 1;
      }
      if (f == base + 1 && t0 != base + 1) {  // nothing new ready, and the next own tile needs more
        __nanosleep(64);
        continue;
      }
      // inclusive values along the run, into incl_sm[pos - base - 1]
      int32_t carry = base_inc;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t pos = base + 1 + j * 32 + lane;
        if (base + 1 + j * 32 >= f) break;
        const uint32_t hi = (uint32_t)(sw[j] >> 32);
        const bool in = pos < f;
        bool seg = in && hi == ((epoch << 2) | F_INC);
        int32_t x = in ? (int32_t)(uint32_t)sw[j] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, x, d);
          const bool sg = __shfl_up_sync(0xffffffffu, seg, d);
          if (lane >= d && !seg) {
            x += y;
            seg = sg;
          }
        }
        if (!seg) x += carry;
        if (in) incl_sm[j * 32 + lane] = x;
        carry = __shfl_sync(0xffffffffu, x, 31);
      }
      __syncwarp();
      // hand out prefixes of own tiles whose predecessors are all in the run
      while (kr < kk) {
        const int64_t t = *reinterpret_cast<volatile int64_t *>(&tid_ring[kr % TR]);
        if (t >= ntiles || t > f) break;
        const int32_t P = t - 1 == base ? base_inc : incl_sm[t - 1 - base - 1];
        if (lane == 0) {
          TRC(3)
          pre_ring[kr % TR] = P;
          mb_arrive(&pref[kr % TR]);
          TRC(4)
          if (t < f) st_relaxed(status + t, tagw(epoch, F_INC, incl_sm[t - base - 1]));
        }
        ++kr;
      }
      if (f - 1 > base) {
        base_inc = incl_sm[f - 1 - base - 1];
        base = f - 1;
      }
      __syncwarp();
    }
  }

  if (LBM != 2 && w > W && w <= W + NLB) {  // ------------------------------ look-back
    const int j = w - (W + 1);
    int64_t prev_t = -1;  // this warp's previous tile and its inclusive value
    int32_t prev_inc = 0;
    for (int64_t k = j;; k += NLB) {
      // the tile id is known at issue; the look-back starts there (EARLY) or
      // once the tile's own aggregate is published
      while (*reinterpret_cast<volatile int64_t *>(&issued) <= k) __nanosleep(32);
      const int64_t t = *reinterpret_cast<volatile int64_t *>(&tid_ring[k % TR]);
      if (t >= ntiles) return;
      if (!EARLY) mb_wait(&folded[k % TR], (uint32_t)((k / TR) & 1));
      if (lane == 0) TRC(3)
      int32_t P = 0;
      if (t > 0) {
        int64_t base = t - 1;
        for (;;) {
          uint64_t sw[8];
          int dstop;
          for (;;) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int64_t idx = base - (jj * 32 + lane);
              sw[jj] = (idx >= 0 && idx != prev_t) ? ld_relaxed(status + idx) : 0;
            }
            dstop = 256;
            bool ok = true;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int64_t idx = base - (jj * 32 + lane);
              const uint32_t hi = (uint32_t)(sw[jj] >> 32);
              const bool stop = idx < 0 || idx == prev_t || hi == ((epoch << 2) | F_INC);
              const unsigned m = __ballot_sync(0xffffffffu, stop);
              if (m && dstop == 256) dstop = jj * 32 + __ffs(m) - 1;
              if (jj * 32 + lane <= dstop && !stop && hi != ((epoch << 2) | F_AGG)) ok = false;
            }
            if (__all_sync(0xffffffffu, ok)) break;
          }
          int32_t part = 0;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int64_t idx = base - (jj * 32 + lane);
            if (jj * 32 + lane <= dstop && idx >= 0) part += idx == prev_t ? prev_inc : (int32_t)(uint32_t)sw[jj];
          }
#pragma unroll
          for (int d = 16; d; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
          P += part;
          if (dstop < 256) break;
          base -= 256;
        }
      }
      if (EARLY) mb_wait(&folded[k % TR], (uint32_t)((k / TR) & 1));
      const int32_t agg = *reinterpret_cast<volatile int32_t *>(&agg_ring[k % TR]);
      if (t > 0 && lane == 0) st_relaxed(status + t, tagw(epoch, F_INC, P + agg));
      prev_t = t;
      prev_inc = P + agg;
      if (lane == 0) {
        pre_ring[k % TR] = P;
        mb_arrive(&pref[k % TR]);
        TRC(4)
      }
      __syncwarp();
    }
  }

  if (w < W) {  // ------------------------------------------------------------ data
    // load(k): wait for use k's stage, copy it into registers, release the
    // stage, fold the warp's rows and publish the warp total; false at the
    // sentinel.  scan(k): wait for use k's prefix, scan the rows, store.
    auto load = [&](int64_t k, uint4 (&v)[R], int64_t &t) -> bool {
      const int s = (int)(k % S);
      mb_wait(&full[s], (uint32_t)((k / S) & 1));
      t = *reinterpret_cast<volatile int64_t *>(&tid_ring[k % TR]);
      if (t >= ntiles) return false;
      const char *st = smem + s * TB + (w * R) * 512 + lane * 16;
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = *reinterpret_cast<const uint4 *>(st + r * 512);
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
      if (w == 0 && lane == 0) TRC(5)
      int32_t a = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) a += (int32_t)v[r].x + (int32_t)v[r].y + (int32_t)v[r].z + (int32_t)v[r].w;
#pragma unroll
      for (int d = 16; d; d >>= 1) a += __shfl_xor_sync(0xffffffffu, a, d);
      if (lane == 0) wt[k % 3][w] = a;
      asm volatile("bar.sync 3, %0;" ::"n"(W * 32) : "memory");
      return true;
    };
    auto scan = [&](int64_t k, const uint4 (&v)[R], int64_t t) {
      int32_t carry = 0;
      for (int i = 0; i < w; ++i) carry += wt[k % 3][i];
      mb_wait(&pref[k % TR], (uint32_t)((k / TR) & 1));
      carry += *reinterpret_cast<volatile int32_t *>(&pre_ring[k % TR]);
      if (w == 0 && lane == 0) TRC(6)
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
      if (w == 0 && lane == 0) TRC(7)
    };
    uint4 va[R], vb[R];
    int64_t ta, tb;
    if (!DB) {
      for (int64_t k = 0;; ++k) {
        if (!load(k, va, ta)) return;
        scan(k, va, ta);
      }
    }
    // two tiles in registers: tile k waits for its prefix while k+1 is
    // already copied out of its stage
    if (!load(0, va, ta)) return;
    for (int64_t k = 0;; k += 2) {
      const bool hb = load(k + 1, vb, tb);
      scan(k, va, ta);
      if (!hb) return;
      const bool ha = load(k + 2, va, ta);
      scan(k + 1, vb, tb);
      if (!ha) return;
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

template <int W, int R, int S, int F, int NLB, int C, int PIECES, int EARLY, bool DB>
int run(int ex, int64_t n, const int32_t *in, int32_t *out, uint64_t *status, unsigned long long *ticket,
        uint32_t epoch, cudaStream_t st, uint64_t *trace = nullptr) {
  constexpr int TB = W * R * 512;
  constexpr int TE = TB / 4;
  if (n % TE) return 3;
  const int64_t ntiles = n / TE;
  auto k0 = ring_scan<W, R, S, F, NLB, C, false, PIECES, EARLY, DB>;
  auto k1 = ring_scan<W, R, S, F, NLB, C, true, PIECES, EARLY, DB>;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, S * TB);
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, S * TB);
    init = true;
  }
  int grid = sms() * C;
  if (grid > ntiles) grid = (int)ntiles;
  (ex ? k1 : k0)<<<grid, (W + 1 + NLB + F) * 32, S * TB, st>>>(in, out, ntiles, status, ticket, epoch, trace);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

}  // namespace

// id: W warps, R rows per warp (512 B), S stages, C CTAs per SM
// id: W data warps, R rows per warp (512 B), S stages, F fold warps, NLB look-back warps, C CTAs per SM,
// bulk pieces, look-back from issue (EARLY) or from landing
#define V(X)                                 \
  X(0, 16, 8, 1, 2, 1, 1, 4, 0, true)        \
  X(1, 16, 8, 3, 2, 1, 1, 4, 0, true)        \
  X(2, 16, 8, 3, 2, 2, 1, 4, 0, true)        \
  X(3, 16, 8, 2, 2, 2, 1, 4, 0, true)        \
  X(4, 16, 4, 2, 2, 1, 1, 2, 0, true)        \
  X(5, 16, 4, 3, 2, 2, 1, 2, 0, true)        \
  X(6, 8, 16, 3, 2, 2, 1, 4, 0, true)        \
  X(7, 16, 8, 1, 2, 1, 1, 4, 2, true)        \
  X(8, 16, 4, 6, 2, 2, 1, 2, 0, true)        \
  X(9, 16, 8, 3, 2, 3, 1, 4, 0, true)

extern "C" int ring_lab(int v, int ex, int64_t n, const void *in, void *out, void *status, void *ticket,
                        uint32_t epoch, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t *i = (const int32_t *)in;
  int32_t *o = (int32_t *)out;
  uint64_t *stt = (uint64_t *)status;
  unsigned long long *tk = (unsigned long long *)ticket;
  switch (v) {
#define C(id, W, R, S, F, NLB, CC, P, E, D) \
  case id: return run<W, R, S, F, NLB, CC, P, E, D>(ex, n, i, o, stt, tk, epoch, s);
    V(C)
#undef C
  }
  return 2;
}
extern "C" int ring_lab_tile_elems(int v) {
  switch (v) {
#define C(id, W, R, S, F, NLB, CC, P, E, D) \
  case id: return W * R * 128;
    V(C)
#undef C
  }
  return 0;
}

extern "C" int ring_lab_trace(int v, int64_t n, const void *in, void *out, void *status, void *ticket, uint32_t epoch,
                              void *trace, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t *i = (const int32_t *)in;
  int32_t *o = (int32_t *)out;
  uint64_t *stt = (uint64_t *)status;
  unsigned long long *tk = (unsigned long long *)ticket;
  switch (v) {
#define C(id, W, R, S, F, NLB, CC, P, E, D) \
  case id: return run<W, R, S, F, NLB, CC, P, E, D>(1, n, i, o, stt, tk, epoch, s, (uint64_t *)trace);
    V(C)
#undef C
  }
  return 2;
}
