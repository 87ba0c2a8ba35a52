// scan_impl.cuh — launch logic of the scans (scan.cu dispatches; the
// super-tile shapes are compiled in separate translation units scan_s.cu,
// scan_m.cu, scan_l.cu so the build runs them in parallel).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "ga_host.h"
#include "scan_kernel.cuh"

namespace ga {
namespace scan_impl {

using namespace scan_detail;

// Super-tile shapes (tools/lab/run_tile_lab.py, profiles/r1_scan_tiles.md):
//   L  24 warps x 32 rows of 512 input bytes (384 KiB per CTA, one CTA per
//      SM): fewest look-back hops, the streaming shape — used when it gives
//      at least L_MIN_TILES tiles (below that the last wave leaves SMs idle);
//   M  32 warps x 8 rows (128 KiB) when that gives at least M_MIN_TILES;
//   S  8 warps (16 for 8-byte T) x 8 rows otherwise: enough tiles to spread
//      a small array over the SMs.
// Every warp keeps 8 rows of 512 bytes in flight in phase 1 (P1U) and
// UNROLL rows in phase 3: 8 for 4-byte types and exclusive int64 at the L
// shape, 4 for the other 8-byte scans, 2 for widened ones, which keeps every
// instance spill-free (ptxas -v) — widened scans 10-14% faster at
// 2^28-2^30 and int64 inclusive 3% faster than with 8 rows and spills
// (tools/lab/ab_scan.py); the look-back
// reads 8 (4 for 8-byte T) predecessors per lane per round trip; warps 1..
// load and locally scan their first phase-3 rows while warp 0 looks back,
// and (L shape) every warp has the TMA unit prefetch its slice of the tile
// 2/7 of a wave ahead (42 ids on 148 SMs) into L2, so the HBM reads of a
// later tile's phase 1 fill the time this SM would otherwise idle in the
// look-back: int32 2^28 415 -> 379 us, 2^30 1540 -> 1398 us (6.1 TB/s), int64
// 2^28 849 -> 802 us (tools/lab/run_tile_lab.py PFV variants,
// profiles/r1_scan_limits.md).
// RG: the register-tile fallback for arrays that are not 16-byte aligned
// (32-byte for a widened output): 256 threads x 16 scalar-loaded items.
enum Shape { SHAPE_S = 0, SHAPE_M = 1, SHAPE_L = 2, SHAPE_RG = 3 };
constexpr int64_t L_MIN_TILES = 256, M_MIN_TILES = 64;
constexpr int UNROLL4 = 8, UNROLL8 = 4, UNROLLW = 2, P1U = 8, DEPTH4 = 8, DEPTH8 = 4;
constexpr int RG_BLOCK = 256, RG_ITEMS = 16, RG_DEPTH = 4;


constexpr int shape_warps(int shape, size_t osz) { return shape == SHAPE_S ? (osz == 8 ? 16 : 8) : shape == SHAPE_M ? 32 : 24; }
constexpr int shape_rows(int shape) { return shape == SHAPE_L ? 32 : 8; }
template <int SHAPE, typename T>
struct ShapeOf {
  static constexpr int WARPS = shape_warps(SHAPE, sizeof(T));
  static constexpr int ROWS = shape_rows(SHAPE);
};

// Host-side shape choice for element sizes (isz in, osz out).
inline int64_t shape_tile(int shape, size_t isz, size_t osz) {
  return (int64_t)shape_warps(shape, osz) * shape_rows(shape) * 512 / (int64_t)isz;
}
inline int choose_shape(int64_t n, size_t isz, size_t osz) {
  if (cdiv(n, shape_tile(SHAPE_L, isz, osz)) >= L_MIN_TILES) return SHAPE_L;
  if (cdiv(n, shape_tile(SHAPE_M, isz, osz)) >= M_MIN_TILES) return SHAPE_M;
  return SHAPE_S;
}

template <int SHAPE, typename T, typename Tin>
constexpr int64_t tile_elems() {
  if constexpr (SHAPE == SHAPE_RG) return (int64_t)RG_BLOCK * RG_ITEMS;
  else return (int64_t)ShapeOf<SHAPE, T>::WARPS * ShapeOf<SHAPE, T>::ROWS * 512 / (int64_t)sizeof(Tin);
}

// Tin != T: the widened scans (int32 -> int64, float -> double; NEXT-2),
// same kernels, the input converted on load; a widened row stores 32 bytes
// per lane (the caller routes outputs that are not 32-byte aligned to RG).
template <int SHAPE, int OP, typename T, typename Tin, bool EXCLUSIVE>
ga_status_t run(int64_t n, const void *in, void *out, const void *carry, int64_t carry_count, void *ws,
                cudaStream_t s) {
  ScanArgs<T, Tin> p = make_args<T, Tin>(n, tile_elems<SHAPE, T, Tin>(), in, out, carry, carry_count, ws);
  if (p.num_tiles > 0x7fffffffLL) return fail(GA_ERR_UNSUPPORTED, "scan: n too large (%lld)", (long long)n);
  const int grid = (int)p.num_tiles;
  if constexpr (SHAPE == SHAPE_RG) {
    launch(scan_reg_kernel<OP, T, Tin, RG_BLOCK, RG_ITEMS, RG_DEPTH, EXCLUSIVE>, grid, RG_BLOCK, 0, s, p);
  } else {
    constexpr int W = ShapeOf<SHAPE, T>::WARPS, R = ShapeOf<SHAPE, T>::ROWS;
    constexpr int D = sizeof(T) == 8 ? DEPTH8 : DEPTH4;
    // exclusive int64 at the L shape fits 8 rows without spilling (and is 3% faster with them)
    constexpr bool ROWS8 = sizeof(T) == 4 || (EXCLUSIVE && SHAPE == SHAPE_L && std::is_integral<T>::value);
    constexpr int U = sizeof(T) != sizeof(Tin) ? UNROLLW : ROWS8 ? UNROLL4 : UNROLL8;
    // L shape: while a tile looks back, its CTA has the TMA unit prefetch the
    // whole input of the tile ~2/7 of a wave ahead into L2 (see the kernel)
    // (not for widened scans: their 2x larger output changes the timing; measured 1-7% slower)
    constexpr int PF = (SHAPE == SHAPE_L && sizeof(T) == sizeof(Tin)) ? R : 0;
    if (PF) p.pf_dist = std::max<int64_t>(1, (int64_t)sm_count() * 2 / 7);
    // 8-byte scans at the L shape: 1 KiB rows (LDG/STG.256, 4 elements per
    // lane per row: half the memory instructions and half the shuffles of
    // the 512-byte rows) when both arrays are 32-byte aligned — 2-5% faster
    // at 2^28-2^30 (profiles/r2_scan.md); same tile, so the same workspace.
    // Widened scans (4-byte in, 8-byte scan) likewise take 1 KiB input rows
    // (2 rows in flight per warp in phase 3, no prefetch): 7-8% faster at
    // 2^28-2^30 (tools/lab/run_wide_lab.py).
    if constexpr (SHAPE == SHAPE_L && sizeof(T) == 8) {
      if ((((uintptr_t)in | (uintptr_t)out) & 31) == 0) {
        constexpr bool WIDE = sizeof(Tin) == 4;
        constexpr int R2 = R / 2, U2 = WIDE ? 2 : 4, P2 = 4, PF2 = WIDE ? 0 : R2;
        if (in == out)
          launch(scan_l2_kernel<OP, T, Tin, W, R2, U2, D, false, EXCLUSIVE, true, P2, PF2, false, 1024>, grid, W * 32,
                 0, s, p, (uint64_t *)nullptr);
        else
          launch(scan_l2_kernel<OP, T, Tin, W, R2, U2, D, true, EXCLUSIVE, true, P2, PF2, false, 1024>, grid, W * 32,
                 0, s, p, (uint64_t *)nullptr);
        count_launch();
        return check_launch("scan_kernel");
      }
    }
    if (in == out)
      launch(scan_l2_kernel<OP, T, Tin, W, R, U, D, false, EXCLUSIVE, true, P1U, PF>, grid, W * 32, 0, s, p,
             (uint64_t *)nullptr);
    else
      launch(scan_l2_kernel<OP, T, Tin, W, R, U, D, true, EXCLUSIVE, true, P1U, PF>, grid, W * 32, 0, s, p,
             (uint64_t *)nullptr);
  }
  count_launch();
  return check_launch("scan_kernel");
}

template <int SHAPE, int OP, typename T, typename Tin>
ga_status_t by_kind(bool ex, int64_t n, const void *in, void *out, const void *carry, int64_t cc, void *ws,
                    cudaStream_t s) {
  return ex ? run<SHAPE, OP, T, Tin, true>(n, in, out, carry, cc, ws, s)
            : run<SHAPE, OP, T, Tin, false>(n, in, out, carry, cc, ws, s);
}

template <int SHAPE, typename T, typename Tin = T>
ga_status_t by_op(ga_op_t op, bool ex, int64_t n, const void *in, void *out, const void *carry, int64_t cc, void *ws,
                  cudaStream_t s) {
  switch (op) {
    case GA_OP_SUM: return by_kind<SHAPE, GA_OP_SUM, T, Tin>(ex, n, in, out, carry, cc, ws, s);
    case GA_OP_MAX: return by_kind<SHAPE, GA_OP_MAX, T, Tin>(ex, n, in, out, carry, cc, ws, s);
    case GA_OP_MIN: return by_kind<SHAPE, GA_OP_MIN, T, Tin>(ex, n, in, out, carry, cc, ws, s);
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad op %d", (int)op);
}

// One shape, every (op, kind, in_dt -> dt) instance; the caller has checked
// the arguments.  Explicitly instantiated once per shape.
template <int SHAPE>
ga_status_t launch_shape(ga_op_t op, bool ex, ga_dtype_t in_dt, ga_dtype_t dt, int64_t n, const void *in, void *out,
                         const void *carry, int64_t cc, void *ws, cudaStream_t s) {
  if (in_dt != dt) {
    if (in_dt == GA_I32 && dt == GA_I64) return by_op<SHAPE, int64_t, int32_t>(op, ex, n, in, out, carry, cc, ws, s);
    if (in_dt == GA_F32 && dt == GA_F64) return by_op<SHAPE, double, float>(op, ex, n, in, out, carry, cc, ws, s);
    return fail(GA_ERR_UNSUPPORTED, "scan %d -> %d not instantiated", (int)in_dt, (int)dt);
  }
  switch (dt) {
    case GA_I32: return by_op<SHAPE, int32_t>(op, ex, n, in, out, carry, cc, ws, s);
    case GA_I64: return by_op<SHAPE, int64_t>(op, ex, n, in, out, carry, cc, ws, s);
    case GA_F32: return by_op<SHAPE, float>(op, ex, n, in, out, carry, cc, ws, s);
    case GA_F64: return by_op<SHAPE, double>(op, ex, n, in, out, carry, cc, ws, s);
    default: break;
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad dtype %d", (int)dt);
}

// The ring scan (scan_ring.cuh, scan_r.cu): 16 data warps x 8 rows of 512 B
// (64 KiB tiles), 3 stages, 2 fold warps; non-widening, 16-byte aligned.
constexpr int RING_W = 16, RING_R = 8, RING_S = 3, RING_F = 2;
// Size window of the ring scan (tools/lab/run_ring_ab.py, same process, back
// to back against the two-touch shapes; profiles/r2_ring.md): from 48 MiB of
// input (int32 32 MiB: even; 64 MiB: -16%) up to
//   4 GiB for 4-byte types (with the one-tile L2 prefetch: 2^28 -8%, 2^30
//        -1 to -3%; 2^31: even to +6%, 2^32-2^33: even to +4%),
//   2 GiB for 8-byte types (1 KiB rows and the prefetch: 2^27 -5 to -9%,
//        2^28 -2 to -5%; 2^29-2^30: -4 to +6%), which needs a 32-byte
//        aligned output (else the two-touch shapes run),
//   any size for widening scans (4-byte in, 8-byte out: -17% at 64 MiB, -7%
//        at 1 GiB, -5% at 4 GiB for SUM; the input arrives at a third of the
//        traffic rate, so the on-chip buffer covers the look-back; MAX within
//        +-1.4%).
constexpr int64_t RING_MIN_BYTES = 48ll << 20, RING_MAX_BYTES4 = 4ll << 30, RING_MAX_BYTES8 = 2ll << 30;
inline bool use_ring(int64_t n, size_t isz, size_t osz, const void *out) {
  const int64_t b = n * (int64_t)isz;
  if (b < RING_MIN_BYTES) return false;
  if (isz != osz) return true;
  if (isz == 8) return b <= RING_MAX_BYTES8 && ((uintptr_t)out & 31) == 0;
  return b <= RING_MAX_BYTES4;
}
ga_status_t launch_ring(ga_op_t op, bool ex, ga_dtype_t in_dt, ga_dtype_t dt, int64_t n, const void *in, void *out,
                        const void *carry, int64_t cc, void *ws, cudaStream_t s);

#define GA_SCAN_INSTANTIATE(SHAPE)                                                                                 \
  template ga_status_t launch_shape<SHAPE>(ga_op_t, bool, ga_dtype_t, ga_dtype_t, int64_t, const void *, void *, \
                                           const void *, int64_t, void *, cudaStream_t);
extern template ga_status_t launch_shape<SHAPE_S>(ga_op_t, bool, ga_dtype_t, ga_dtype_t, int64_t, const void *,
                                                  void *, const void *, int64_t, void *, cudaStream_t);
extern template ga_status_t launch_shape<SHAPE_M>(ga_op_t, bool, ga_dtype_t, ga_dtype_t, int64_t, const void *,
                                                  void *, const void *, int64_t, void *, cudaStream_t);
extern template ga_status_t launch_shape<SHAPE_L>(ga_op_t, bool, ga_dtype_t, ga_dtype_t, int64_t, const void *,
                                                  void *, const void *, int64_t, void *, cudaStream_t);
extern template ga_status_t launch_shape<SHAPE_RG>(ga_op_t, bool, ga_dtype_t, ga_dtype_t, int64_t, const void *,
                                                   void *, const void *, int64_t, void *, cudaStream_t);

}  // namespace scan_impl
}  // namespace ga
