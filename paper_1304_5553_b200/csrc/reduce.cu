// reduce.cu — ReductionKernel-style map-reduce (§3.2.5):
// "evaluating an element-wise expression ahead of reduction" (463-467), a
// reduction expression of a and b with its neutral element (479-485), and a
// result that is "a GPUArray scalar still residing on the GPU" (489-492).
//
// Single pass, one launch, HBM-bound (4 B/elt fp32 sum/norm2, 8 B/elt dot):
//   1. map + accumulate over a one-shot grid: CTA b owns the contiguous chunk
//      of RED_BLOCK*UNROLL 32-byte vectors starting at b*RED_BLOCK*UNROLL
//      (the grid is capped at RED_MAX_PARTIALS CTAs, beyond which chunks
//      repeat with that stride); each thread keeps one accumulator per lane
//      of a 256-bit vector (8 for fp32) and loads all UNROLL vectors per
//      input before using any (LDG.256, L1 bypassed); scalar head/tail for
//      the unaligned ends; out-of-range work contributes the neutral element
//      (one-shot grids beat a persistent grid-stride wave by ~4%,
//      tools/lab/red_lab.cu; the CTA shape is from red_shape_lab.cu);
//   2. fixed-order lane tree -> warp xor-butterfly -> per-warp partial in
//      shared memory -> warp 0 folds the block partial;
//   3. single-pass finish, two levels (red_detail::grid_finish): a block
//      publishes its partial into a slot tagged with the call's epoch and
//      exits (no fence, no atomic); the last block of each group of 128
//      waits for its group's slots and folds them in index order; the last
//      block of the grid folds the group partials in order, writes *out and
//      advances the epoch (no second launch, no host sync, no memset
//      between calls).
// Deterministic for a given (n, device): the grid depends on n, the finish's
// group size also on the device's SM count (make_finish), and every fold
// order above is fixed by those two.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "ga_device.cuh"
#include "ga_host.h"
#include "reduce_kernel.cuh"

namespace ga {
namespace {

using namespace red_detail;

// Tuned CTA shape (tools/lab/red_shape_lab.cu): 256 threads, 8 vectors in
// flight per thread (UNROLL 8, or 4 per input for x*y), at least 4 CTAs per
// SM (<= 64 registers): 7.04 / 7.22 TB/s sum / dot at n = 2^28 and 6.2 / 6.7
// at 2^26, against 6.81 / 6.94 and 5.9 / 6.4 for 512 threads x 4.
constexpr int RED_BLOCK = 256, RED_MINB = 4;

template <typename Tin, typename Tacc, int OP, int MAP>
ga_status_t run(int64_t n, const void *x, const void *y, void *out, void *ws, const Exchange &xg, cudaStream_t s) {
  if (n == 0 && xg.world == 0) {
    launch(neutral_kernel<Tacc, OP>, 1, 1, 0, s, static_cast<Tacc *>(out));
    count_launch();
    return check_launch("neutral_kernel");
  }
  constexpr int VEC = 32 / sizeof(Tin);
  // Vectors in flight per thread: 8 (4 per input for x*y); half of that
  // where the per-vector work needs more registers — widening accumulators,
  // integer products, MAX/MIN over a product (guarded, no neutral fill) —
  // so that the instances stay within the 64 registers of 4 CTAs/SM
  // without spilling (ptxas -v: 0 bytes for every instance).
  constexpr bool WIDEN = sizeof(Tacc) > sizeof(Tin);
  constexpr bool INT_PRODUCT = !is_fp<Tacc>() && MAP != GA_MAP_ID;
  constexpr int DIV = (WIDEN || (INT_PRODUCT && sizeof(Tacc) == 8)) ? 4
                      : (INT_PRODUCT || (OP != GA_OP_SUM && MAP != GA_MAP_ID)) ? 2 : 1;
  constexpr int UNROLL = std::max(1, ((MAP == GA_MAP_MUL || MAP == GA_MAP_CONJ_MUL) ? 4 : 8) / DIV);
  RedArgs<Tin, Tacc> p;
  p.n = n;
  p.x = static_cast<const Tin *>(x);
  p.y = static_cast<const Tin *>(y);
  p.out = static_cast<Tacc *>(out);
  p.xg = xg;

  const uintptr_t phase = (uintptr_t)x & 31;
  constexpr bool HAS_Y = MAP == GA_MAP_MUL || MAP == GA_MAP_CONJ_MUL;
  const bool coaligned = (!HAS_Y || ((uintptr_t)y & 31) == phase) && (phase % sizeof(Tin)) == 0;
  if (coaligned) {
    p.head = std::min<int64_t>(n, (int64_t)(((32 - phase) & 31) / sizeof(Tin)));
    p.nvec = (n - p.head) / VEC;
  } else {
    p.head = n;
    p.nvec = 0;
  }
  auto kern = reduce_kernel<Tin, Tacc, OP, MAP, UNROLL, RED_BLOCK, RED_MINB>;
  // one CTA per chunk of RED_BLOCK*UNROLL vectors (or RED_BLOCK scalars on
  // the unaligned path), capped at RED_MAX_PARTIALS
  const int64_t units = coaligned ? cdiv(std::max<int64_t>(p.nvec, 1), (int64_t)RED_BLOCK * UNROLL) : cdiv(n, RED_BLOCK);
  const int grid = (int)std::max<int64_t>(std::min<int64_t>(units, RED_MAX_PARTIALS), 1);
  p.fin = make_finish(ws, grid, RED_MINB);
  launch(kern, grid, RED_BLOCK, 0, s, p);
  count_launch();
  return check_launch("reduce_kernel");
}

template <typename Tin, typename Tacc, int OP>
ga_status_t by_map(ga_map_t map, int64_t n, const void *x, const void *y, void *out, void *ws, const Exchange &xg,
                   cudaStream_t s) {
  switch (map) {
    case GA_MAP_ID: return run<Tin, Tacc, OP, GA_MAP_ID>(n, x, y, out, ws, xg, s);
    case GA_MAP_MUL:
    case GA_MAP_CONJ_MUL:  // conj(x) == x for real x
      return run<Tin, Tacc, OP, GA_MAP_MUL>(n, x, y, out, ws, xg, s);
    case GA_MAP_SQUARE: return run<Tin, Tacc, OP, GA_MAP_SQUARE>(n, x, y, out, ws, xg, s);
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "bad map %d", (int)map);
}

// Complex SUM: x | x*y | conj(x)*y into the complex type; |x|^2 into the real one.
template <typename C, typename R>
ga_status_t complex_sum(ga_map_t map, ga_dtype_t out_dt, ga_dtype_t cdt, ga_dtype_t rdt, int64_t n, const void *x,
                        const void *y, void *out, void *ws, const Exchange &xg, cudaStream_t s) {
  if (map == GA_MAP_SQUARE) {
    if (out_dt != rdt) return fail(GA_ERR_UNSUPPORTED, "complex |x|^2 sums into the real type");
    return run<C, R, GA_OP_SUM, GA_MAP_SQUARE>(n, x, y, out, ws, xg, s);
  }
  if (out_dt != cdt) return fail(GA_ERR_UNSUPPORTED, "complex SUM needs out_dt == in_dt");
  switch (map) {
    case GA_MAP_ID: return run<C, C, GA_OP_SUM, GA_MAP_ID>(n, x, y, out, ws, xg, s);
    case GA_MAP_MUL: return run<C, C, GA_OP_SUM, GA_MAP_MUL>(n, x, y, out, ws, xg, s);
    case GA_MAP_CONJ_MUL: return run<C, C, GA_OP_SUM, GA_MAP_CONJ_MUL>(n, x, y, out, ws, xg, s);
    default: break;
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "bad map %d", (int)map);
}

template <typename T, int OP>
ga_status_t maxmin(ga_map_t map, int64_t n, const void *x, const void *y, void *out, void *ws, const Exchange &xg,
                   cudaStream_t s) {
  return by_map<T, T, OP>(map, n, x, y, out, ws, xg, s);
}

}  // namespace

size_t reduce_workspace_bytes() { return RED_WS_BYTES; }  // up to c128 partials

ga_status_t launch_reduce(ga_op_t op, ga_map_t map, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                          const void *x, const void *y, void *out, void *ws, const Exchange &xg, cudaStream_t s) {
  if (in_dt == GA_C64 || in_dt == GA_C128) {
    if (op != GA_OP_SUM) return fail(GA_ERR_UNSUPPORTED, "MAX/MIN are not defined for complex numbers");
    if (in_dt == GA_C64) return complex_sum<c64, float>(map, out_dt, GA_C64, GA_F32, n, x, y, out, ws, xg, s);
    return complex_sum<c128, double>(map, out_dt, GA_C128, GA_F64, n, x, y, out, ws, xg, s);
  }
  if (op == GA_OP_SUM) {
    if (in_dt == GA_F32 && out_dt == GA_F32) return by_map<float, float, GA_OP_SUM>(map, n, x, y, out, ws, xg, s);
    if (in_dt == GA_F32 && out_dt == GA_F64) return by_map<float, double, GA_OP_SUM>(map, n, x, y, out, ws, xg, s);
    if (in_dt == GA_F64 && out_dt == GA_F64) return by_map<double, double, GA_OP_SUM>(map, n, x, y, out, ws, xg, s);
    if (in_dt == GA_I32 && out_dt == GA_I32) return by_map<int32_t, int32_t, GA_OP_SUM>(map, n, x, y, out, ws, xg, s);
    if (in_dt == GA_I32 && out_dt == GA_I64) return by_map<int32_t, int64_t, GA_OP_SUM>(map, n, x, y, out, ws, xg, s);
    if (in_dt == GA_I64 && out_dt == GA_I64) return by_map<int64_t, int64_t, GA_OP_SUM>(map, n, x, y, out, ws, xg, s);
    return fail(GA_ERR_UNSUPPORTED, "SUM %d -> %d not instantiated", (int)in_dt, (int)out_dt);
  }
  if (in_dt != out_dt) return fail(GA_ERR_UNSUPPORTED, "MAX/MIN need out_dt == in_dt");
  if (op == GA_OP_MAX) {
    switch (in_dt) {
      case GA_F32: return maxmin<float, GA_OP_MAX>(map, n, x, y, out, ws, xg, s);
      case GA_F64: return maxmin<double, GA_OP_MAX>(map, n, x, y, out, ws, xg, s);
      case GA_I32: return maxmin<int32_t, GA_OP_MAX>(map, n, x, y, out, ws, xg, s);
      case GA_I64: return maxmin<int64_t, GA_OP_MAX>(map, n, x, y, out, ws, xg, s);
      default: break;
    }
  } else if (op == GA_OP_MIN) {
    switch (in_dt) {
      case GA_F32: return maxmin<float, GA_OP_MIN>(map, n, x, y, out, ws, xg, s);
      case GA_F64: return maxmin<double, GA_OP_MIN>(map, n, x, y, out, ws, xg, s);
      case GA_I32: return maxmin<int32_t, GA_OP_MIN>(map, n, x, y, out, ws, xg, s);
      case GA_I64: return maxmin<int64_t, GA_OP_MIN>(map, n, x, y, out, ws, xg, s);
      default: break;
    }
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "bad op %d", (int)op);
}

}  // namespace ga
