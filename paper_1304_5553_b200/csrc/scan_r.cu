// scan_r.cu — the ring (single-touch) scan for mid-size arrays (see
// scan_ring.cuh), every (op, kind, dtype) instance; scan.cu dispatches.
#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_impl.cuh"
#include "scan_ring.cuh"

namespace ga {
namespace scan_impl {

namespace {
using namespace scan_detail;

// Q: bulk loads in flight per CTA, PFN: tile ids drawn ahead and prefetched
// into L2, H: 16-byte chunks per lane per warp row (0 / -1 = the product
// choice).  Non-widening scans: one bulk load in flight (the next id is
// drawn once the previous load has landed, which narrows the spread of
// landing times the look-back waits on) plus one id drawn ahead whose input
// the producer prefetches into L2, so the HBM read of the next tile overlaps
// and its bulk copy hits L2 — int32 2^26 -10%, 2^28 -8%, 2^30 -1 to -3%
// against the two-touch L shape; 8-byte types also take 1 KiB rows (32
// bytes per lane: half the 64-bit warp scans per element; the output must be
// 32-byte aligned) — int64 -5 to -9% at 2^24-2^27 against the 512-byte-row
// ring, and ahead of the L shape up to 2^28.  Widening scans: all S stages
// in flight, no prefetch, 512-byte rows (neither knob helped them).
// tools/lab/run_ring_ab.py cfg, profiles/r2_ring.md.
template <int OP, typename T, typename Tin, bool EX, int W = RING_W, int R0 = 0, int S = RING_S, int F = RING_F,
          int Q0 = 0, int PFN0 = -1, int H0 = 0>
ga_status_t ring_run(int64_t n, const void *in, void *out, const void *carry, int64_t cc, void *ws, cudaStream_t s) {
  constexpr bool WIDEN = sizeof(T) != sizeof(Tin);
  constexpr int H = H0 > 0 ? H0 : (!WIDEN && sizeof(T) == 8) ? 2 : 1;
  constexpr int R = R0 > 0 ? R0 : RING_R / H;  // 64 KiB tiles
  constexpr int Q = Q0 > 0 ? Q0 : WIDEN ? S : 1;
  constexpr int PFN = PFN0 >= 0 ? PFN0 : WIDEN ? 0 : 1;
  constexpr int64_t TE = (int64_t)W * R * 512 * H / (int64_t)sizeof(Tin);
  constexpr size_t SMEM = (size_t)S * W * R * 512 * H;
  auto k = scan_ring_kernel<OP, T, Tin, W, R, S, F, EX, Q, PFN, H>;
  const cudaError_t attr = allow_dyn_smem((const void *)k, SMEM);
  if (attr != cudaSuccess) return fail(GA_ERR_CUDA, "scan (ring): %s", cudaGetErrorString(attr));
  ScanArgs<T, Tin> p = make_args<T, Tin>(n, TE, in, out, carry, cc, ws);
  const int64_t grid = std::min<int64_t>(sm_count(), p.num_tiles);
  launch(k, (int)grid, ring_threads<W, F>(), SMEM, s, p);
  count_launch();
  return check_launch("scan_ring_kernel");
}

template <typename T, typename Tin = T>
ga_status_t ring_by_op(ga_op_t op, bool ex, int64_t n, const void *in, void *out, const void *carry, int64_t cc,
                       void *ws, cudaStream_t s) {
  switch (op) {
    case GA_OP_SUM:
      return ex ? ring_run<GA_OP_SUM, T, Tin, true>(n, in, out, carry, cc, ws, s)
                : ring_run<GA_OP_SUM, T, Tin, false>(n, in, out, carry, cc, ws, s);
    case GA_OP_MAX:
      return ex ? ring_run<GA_OP_MAX, T, Tin, true>(n, in, out, carry, cc, ws, s)
                : ring_run<GA_OP_MAX, T, Tin, false>(n, in, out, carry, cc, ws, s);
    case GA_OP_MIN:
      return ex ? ring_run<GA_OP_MIN, T, Tin, true>(n, in, out, carry, cc, ws, s)
                : ring_run<GA_OP_MIN, T, Tin, false>(n, in, out, carry, cc, ws, s);
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad op %d", (int)op);
}
}  // namespace

ga_status_t launch_ring(ga_op_t op, bool ex, ga_dtype_t in_dt, ga_dtype_t dt, int64_t n, const void *in, void *out,
                        const void *carry, int64_t cc, void *ws, cudaStream_t s) {
  if (in_dt != dt) {
    if (in_dt == GA_I32 && dt == GA_I64) return ring_by_op<int64_t, int32_t>(op, ex, n, in, out, carry, cc, ws, s);
    if (in_dt == GA_F32 && dt == GA_F64) return ring_by_op<double, float>(op, ex, n, in, out, carry, cc, ws, s);
    return fail(GA_ERR_UNSUPPORTED, "scan %d -> %d not instantiated", (int)in_dt, (int)dt);
  }
  switch (dt) {
    case GA_I32: return ring_by_op<int32_t>(op, ex, n, in, out, carry, cc, ws, s);
    case GA_I64: return ring_by_op<int64_t>(op, ex, n, in, out, carry, cc, ws, s);
    case GA_F32: return ring_by_op<float>(op, ex, n, in, out, carry, cc, ws, s);
    case GA_F64: return ring_by_op<double>(op, ex, n, in, out, carry, cc, ws, s);
    default: break;
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad dtype %d", (int)dt);
}

}  // namespace scan_impl
}  // namespace ga
