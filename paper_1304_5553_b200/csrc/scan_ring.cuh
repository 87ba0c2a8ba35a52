// scan_ring.cuh — the single-touch "ring" scan (§3.2.6;
// scan expressions of P:479-485), used by scan.cu for 16-byte aligned scans
// of 48 MiB .. 4 GiB (4-byte) / 2 GiB (8-byte) of input and for widening
// scans from 48 MiB (scan_impl.cuh use_ring; profiles/r2_ring.md).
//
// Persistent CTAs, one per SM, draw 64 KiB tiles from the workspace ticket
// (the same {epoch | counter} word, status layout and look-back as the
// two-touch kernel), so every HBM byte is read once and written once:
//   warp W       producer: draws tile ids and fills a ring of S shared-memory
//                stages with TMA bulk copies (cp.async.bulk, mbarrier); for
//                non-widening scans it keeps one copy in flight and draws one
//                id ahead whose input it prefetches into L2;
//   warps W+2..  fold: fold each stage as it lands and publish the tile's
//                AGGREGATE at once (tile 0: its INCLUSIVE value with the
//                carry-in), so no aggregate waits behind a look-back;
//   warp W+1     look-back: the decoupled look-back of scan_kernel.cuh for
//                each tile in turn, publishes INCLUSIVE, hands the prefix on;
//   warps 0..W-1 data: copy a landed stage into registers and release it at
//                once, fold their rows, wait for the tile's prefix, scan the
//                rows and store them (512-byte rows; 1 KiB for 8-byte types).
//                They hold TWO tiles: tile k waits for its prefix while tile
//                k+1 is already out of its stage, so the stages keep
//                streaming.
// Per-use values (tile id, aggregate, prefix and their mbarriers) live in
// rings of TR slots, so a role running ahead never overwrites what a slower
// one still needs.  Against the two-touch kernel: int32 2^26 -10%, 2^28 -8%
// (336-343 us, 91% of the 1:1 copy), 2^30 -1 to -3%; int64 2^27 -5 to -9%.
// Beyond the window the L2-buffered two-touch kernel is as fast or faster:
// a tile's prefix arrives ~8-10 us after it lands (it needs every earlier
// tile's aggregate), and the per-SM buffer of stages, registers and one
// prefetched tile only covers that up to a few GiB.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_kernel.cuh"

namespace ga {
namespace scan_detail {
namespace ring {

__device__ __forceinline__ void mb_init(uint64_t *b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Wait for the phase of parity ph; a phase that never completes (a broken
// invariant) traps after 10 s instead of hanging the device.
__device__ __forceinline__ void mb_wait(const uint64_t *b, uint32_t ph) {
  uint32_t done = 0, spins = 0;
  uint64_t t0 = 0;
  while (true) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(smem_u32(b)), "r"(ph)
                 : "memory");
    if (done) return;
    if ((++spins & 255u) == 0) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 10000000000ull) __trap();
    }
  }
}

constexpr int TR = 16;  // ring slots of per-use values

}  // namespace ring

template <int W, int F>
constexpr int ring_threads() {
  return (W + 2 + F) * 32;
}

// MAXQ: bulk loads in flight per CTA (<= S): the producer draws the next
// tile only once the load MAXQ uses back has landed.
// Tin != T: the widening scans (int32 -> int64, float -> double), the input
// converted where it is folded; a row then stores 32 bytes per lane.
// PFN: tile ids drawn this many uses ahead, their input prefetched into L2
// (cp.async.bulk.prefetch.L2) so that the stage's bulk copy later hits L2.
// H: 16-byte chunks per lane per warp row (1: 512-byte rows; 2: 1 KiB rows,
// 32 bytes per lane — half the warp scans per element, 32-byte stores).
template <int OP, typename T, typename Tin, int W, int R, int S, int F, bool EXCLUSIVE, int MAXQ = S, int PFN = 0,
          int H = 1>
__global__ void __launch_bounds__(ring_threads<W, F>(), 1) scan_ring_kernel(ScanArgs<T, Tin> p) {
  pdl_enter();
  using O = Op<OP, T>;
  using namespace ring;
  constexpr int E = 16 / (int)sizeof(Tin);  // elements per 16-byte chunk
  constexpr int EL = E * H;                  // elements per lane per warp row
  constexpr int RB = 512 * H;                // input bytes per warp row
  constexpr int ROW = 32 * EL;
  constexpr int TB = W * R * RB;  // tile input bytes
  constexpr int64_t TE = TB / (int64_t)sizeof(Tin);
  constexpr bool WIDEN = sizeof(T) != sizeof(Tin);
  static_assert(!WIDEN || (sizeof(T) == 8 && sizeof(Tin) == 4), "widening is 4 -> 8 bytes");
  constexpr int PIECES = 4, PB = TB / PIECES;  // bulk copies per stage
  constexpr int DEPTH = sizeof(T) == 8 ? 4 : 8;
  static_assert(TR >= S + 3, "ring too short for the stages");
  static_assert(W <= 32 && F <= 32, "warp counts");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[S], empty[S], folded[TR], pref[TR];
  __shared__ int64_t tid_ring[TR];
  __shared__ int64_t issued;
  __shared__ T agg_ring[TR], pre_ring[TR];
  __shared__ T wt[3][W];
  __shared__ T ft[F];
  __shared__ uint32_t s_epoch, s_first;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T neutral = O::neutral();
  const int64_t nt = p.num_tiles;
  // every CTA draws until its first id >= nt, so a call draws exactly
  // nt + gridDim.x ids; the last draw resets the counter and bumps the epoch
  auto draw = [&](uint32_t &epoch) -> int64_t {
    const unsigned long long old = atomicAdd(p.ticket, 1ull);
    const uint32_t ctr = (uint32_t)old;
    epoch = (uint32_t)(old >> 32) & EPOCH_MASK;
    if ((int64_t)ctr == nt + gridDim.x - 1) *p.ticket = (unsigned long long)((epoch + 1u) & EPOCH_MASK) << 32;
    return (int64_t)ctr;
  };
  // input bytes of tile t moved by the bulk copies (a multiple of 16; the
  // ragged tail beyond them is read element by element)
  auto bulk_bytes = [&](int64_t t) -> int64_t {
    const int64_t b = (p.n - t * TE) * (int64_t)sizeof(Tin);
    return b >= TB ? TB : (b & ~(int64_t)15);
  };
  // 16 bytes (E elements) at byte offset `off` of tile t: from the stage, or
  // (ragged tile, past the bulk bytes) from global memory, neutral past n
  auto chunk = [&](const unsigned char *stage, int64_t t, int off, int64_t bulk) -> uint4 {
    if (off + 16 <= bulk) return *reinterpret_cast<const uint4 *>(stage + off);
    const int64_t i = t * TE + off / (int)sizeof(Tin);
    Tin e[E];
#pragma unroll
    for (int k = 0; k < E; ++k) e[k] = i + k < p.n ? p.in[i + k] : Op<OP, Tin>::neutral();
    return Chunk<Tin>::pack(e);
  };
  // the E input elements of a raw 16-byte chunk, converted to T
  auto unpack = [&](const uint4 &raw, T (&v)[E]) {
    Tin e[E];
    Chunk<Tin>::unpack(raw, e);
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = (T)e[k];
  };

  if (threadIdx.x == 0) {
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
    uint32_t e;
    s_first = (uint32_t)draw(e);
    s_epoch = e;
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;

  if (warp == W) {  // ---------------------------------------------------------- producer
    if (lane != 0) return;
    const uint64_t drop = l2::policy_evict_first();
    const uint64_t keep = l2::policy_evict_last();
    // FIFO of ids drawn ahead (PFN > 0): the id handed out next plus up to
    // PFN more, each prefetched into L2 when drawn; drawing stops after the
    // CTA's one id past the last tile.  Fixed-index register array.
    int64_t ahead[PFN + 1];
    int nahead = 0;
    bool more = true;
    auto next_id = [&](bool first) -> int64_t {
      uint32_t e;
      if constexpr (PFN == 0) {
        return first ? (int64_t)s_first : draw(e);
      } else {
        if (first) {
          ahead[0] = (int64_t)s_first;
          nahead = 1;
          more = (int64_t)s_first < nt;
        }
        while (more && nahead < PFN + 1) {
          const int64_t d = draw(e);
          more = d < nt;
          if (more && bulk_bytes(d) > 0)
            asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(
                             reinterpret_cast<const unsigned char *>(p.in) + d * (int64_t)TB),
                         "r"((uint32_t)bulk_bytes(d)), "l"(keep)
                         : "memory");
#pragma unroll
          for (int i = 0; i <= PFN; ++i)
            if (i == nahead) ahead[i] = d;
          ++nahead;
        }
        const int64_t t = ahead[0];
#pragma unroll
        for (int i = 0; i < PFN; ++i) ahead[i] = ahead[i + 1];
        --nahead;
        return t;
      }
    };
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      if (k >= S) mb_wait(&empty[s], (uint32_t)((k / S - 1) & 1));
      if (MAXQ < S && k >= MAXQ) mb_wait(&full[(k - MAXQ) % S], (uint32_t)(((k - MAXQ) / S) & 1));
      const int64_t t = next_id(k == 0);
      tid_ring[k % TR] = t;
      __threadfence_block();
      *reinterpret_cast<volatile int64_t *>(&issued) = k + 1;
      if (t >= nt) {
        mb_arrive(&full[s]);  // the sentinel wakes the data and fold warps, who stop
        return;
      }
      const int64_t bulk = bulk_bytes(t);
      if (bulk == 0) {
        mb_arrive(&full[s]);
        continue;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                   "r"((uint32_t)bulk)
                   : "memory");
      const unsigned char *src = reinterpret_cast<const unsigned char *>(p.in) + t * (int64_t)TB;
#pragma unroll
      for (int i = 0; i < PIECES; ++i) {
        const int64_t off = (int64_t)i * PB;
        if (off < bulk) {
          const uint32_t sz = (uint32_t)(bulk - off < PB ? bulk - off : PB);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
              "[%3], %4;" ::"r"(smem_u32(smem + s * TB + off)),
              "l"(src + off), "r"(sz), "r"(smem_u32(&full[s])), "l"(drop)
              : "memory");
        }
      }
    }
  }

  if (warp >= W + 2) {  // -------------------------------------------------------- fold
    const int f = warp - (W + 2);
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      mb_wait(&full[s], (uint32_t)((k / S) & 1));
      const int64_t t = *reinterpret_cast<volatile int64_t *>(&tid_ring[k % TR]);
      if (t >= nt) return;
      const unsigned char *stage = smem + s * TB;
      const int64_t bulk = bulk_bytes(t);
      T a = neutral;
      if (bulk == TB) {
#pragma unroll 8
        for (int i = 0; i < TB / (F * 512); ++i) {
          T e[E];
          unpack(*reinterpret_cast<const uint4 *>(stage + (i * F * 32 + f * 32 + lane) * 16), e);
#pragma unroll
          for (int q = 0; q < E; ++q) a = O::fold(a, e[q]);
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < TB / (F * 512); ++i) {
          T e[E];
          unpack(chunk(stage, t, (i * F * 32 + f * 32 + lane) * 16, bulk), e);
#pragma unroll
          for (int q = 0; q < E; ++q) a = O::fold(a, e[q]);
        }
      }
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
      a = warp_fold<OP, T>(a);
      if constexpr (F > 1) {
        if (lane == 0) ft[f] = a;
        asm volatile("bar.sync 2, %0;" ::"n"(F * 32) : "memory");
        if (f == 0) {
          a = ft[0];
          for (int i = 1; i < F; ++i) a = O::fold(a, ft[i]);
        }
        asm volatile("bar.sync 2, %0;" ::"n"(F * 32) : "memory");
      }
      if (f == 0 && lane == 0) {
        if (t == 0) p.status.publish(0, epoch, FLAG_INCLUSIVE, O::fold(carry_in<OP, T, Tin>(p), a));
        else p.status.publish(t, epoch, FLAG_AGGREGATE, a);
        agg_ring[k % TR] = a;
        mb_arrive(&folded[k % TR]);
      }
    }
  }

  if (warp == W + 1) {  // ----------------------------------------------------- look-back
    for (int64_t k = 0;; ++k) {
      while (*reinterpret_cast<volatile int64_t *>(&issued) <= k) __nanosleep(32);
      __syncwarp();
      const int64_t t = *reinterpret_cast<volatile int64_t *>(&tid_ring[k % TR]);
      if (t >= nt) return;
      mb_wait(&folded[k % TR], (uint32_t)((k / TR) & 1));  // our AGGREGATE is out
      T P;
      if (t == 0) {
        P = carry_in<OP, T, Tin>(p);
      } else {
        P = look_back<OP, T, DEPTH>(p.status, t, epoch);
        if (lane == 0) p.status.publish(t, epoch, FLAG_INCLUSIVE, O::fold(P, agg_ring[k % TR]));
      }
      if (lane == 0) {
        pre_ring[k % TR] = P;
        mb_arrive(&pref[k % TR]);
      }
      __syncwarp();
    }
  }

  if (warp < W) {  // -------------------------------------------------------------- data
    // load(k): wait for use k's stage, copy this warp's R rows into registers,
    // release the stage, fold the rows into wt; false at the sentinel.
    auto load = [&](int64_t k, uint4 (&v)[R][H], int64_t &t) -> bool {
      const int s = (int)(k % S);
      mb_wait(&full[s], (uint32_t)((k / S) & 1));
      t = *reinterpret_cast<volatile int64_t *>(&tid_ring[k % TR]);
      if (t >= nt) return false;
      const unsigned char *stage = smem + s * TB;
      const int64_t bulk = bulk_bytes(t);
      const int off0 = warp * R * RB + lane * 16 * H;
      if (bulk == TB) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int h = 0; h < H; ++h) v[r][h] = *reinterpret_cast<const uint4 *>(stage + off0 + r * RB + h * 16);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int h = 0; h < H; ++h) v[r][h] = chunk(stage, t, off0 + r * RB + h * 16, bulk);
      }
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
      T a = neutral;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int h = 0; h < H; ++h) {
          T e[E];
          unpack(v[r][h], e);
#pragma unroll
          for (int q = 0; q < E; ++q) a = O::fold(a, e[q]);
        }
      a = warp_fold<OP, T>(a);
      if (lane == 0) wt[k % 3][warp] = a;
      asm volatile("bar.sync 3, %0;" ::"n"(W * 32) : "memory");
      return true;
    };
    // scan(k): wait for use k's prefix, scan the rows in order, store.
    auto scan = [&](int64_t k, const uint4 (&v)[R][H], int64_t t) {
      const uint64_t drop = l2::policy_evict_first();
      mb_wait(&pref[k % TR], (uint32_t)((k / TR) & 1));
      T carry = pre_ring[k % TR];
      for (int i = 0; i < warp; ++i) carry = O::fold(carry, wt[k % 3][i]);
      const int64_t i0 = t * TE + (int64_t)warp * R * ROW + lane * EL;
      const bool full_tile = (t + 1) * TE <= p.n;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        T e[EL], o[EL];
#pragma unroll
        for (int h = 0; h < H; ++h) {
          T c[E];
          unpack(v[r][h], c);
#pragma unroll
          for (int q = 0; q < E; ++q) e[h * E + q] = c[q];
        }
#pragma unroll
        for (int q = 1; q < EL; ++q) e[q] = O::fold(e[q - 1], e[q]);
        const T x = warp_inclusive<OP, T>(e[EL - 1], lane);
        const T cb = O::fold(carry, warp_exclusive_of<OP, T>(x, lane));
        carry = O::fold(carry, __shfl_sync(0xffffffffu, x, 31));
#pragma unroll
        for (int q = 0; q < EL; ++q) {
          if constexpr (EXCLUSIVE) o[q] = q == 0 ? cb : O::fold(cb, e[q - 1]);
          else o[q] = O::fold(cb, e[q]);
        }
        const int64_t i = i0 + (int64_t)r * ROW;
        if (full_tile || i + EL <= p.n) {
          constexpr int OB = EL * (int)sizeof(T);  // output bytes per lane: 16, 32 or 64
          if constexpr (OB == 16) {
            l2::stg128_hint(p.out + i, Chunk<T>::pack(o), drop);
          } else {  // 32-byte stores (the caller guarantees a 32-byte aligned output)
            constexpr int EPV = 32 / (int)sizeof(T);
#pragma unroll
            for (int g = 0; g < OB / 32; ++g) {
              V32 w;
#pragma unroll
              for (int q = 0; q < EPV; ++q) vset<T>(w, q, o[g * EPV + q]);
              l2::stg256v_hint(p.out + i + g * EPV, w, drop);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < EL; ++q)
            if (i + q < p.n) p.out[i + q] = o[q];
        }
      }
    };
    uint4 va[R][H], vb[R][H];
    int64_t ta, tb;
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

}  // namespace scan_detail
}  // namespace ga
