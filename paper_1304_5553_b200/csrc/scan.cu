// scan.cu — parallel prefix sum (§3.2.6: "GPU-based
// parallel prefix sums (also known as `parallel scan')") with the scan
// expressions "+", max, min (the reduction expressions of P:479-485) over
// int32 / int64 (wrapping, R4/R14) and float / double (R22).
//
// One launch, decoupled look-back across super-tiles (BASELINE.json
// north_star), HBM traffic 1 read + 1 write per element when the super-tiles
// in flight stay L2-resident (scan_l2_kernel in scan_kernel.cuh):
//   - CTA draws {epoch, super-tile id} with one 64-bit atomic (ids in CTA
//     start order, so every predecessor is already running);
//   - phase 1 streams its 384 KiB super-tile from HBM (each of 24 warps its
//     own 16 KiB slice, 8 x 512-byte rows in flight, L2 evict_last) and sums
//     it; the AGGREGATE is published as soon as the sum is known;
//   - phase 2: warp 0 looks back over 256 predecessors per round trip,
//     stopping at the nearest INCLUSIVE, and publishes INCLUSIVE; meanwhile
//     the other warps already load and locally scan their first 8 rows;
//   - phase 3 re-reads the slice (L2 hit, evict_first), scans it row by row
//     (in-chunk serial scan + warp shuffle scan) and stores 512 B per warp
//     instruction.
// Look-back status words carry the call's epoch, so the workspace is zeroed
// once and never again; the CTA drawing the last id resets the counter.
// Tile 0's exclusive prefix is the carry-in c = sum(carry[0..carry_count)),
// which is how a sharded scan injects the totals of earlier shards.
// tools/lab/scan_lab.cu keeps the alternatives that were measured against
// this one (register-tiled single-touch, TMA-staged, warp-specialized).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ga_host.h"
#include "scan_kernel.cuh"

namespace ga {
namespace {

using namespace scan_detail;

// Tuned super-tile shape (tools/lab/run_scan_lab.py): 24 warps x 32 rows of
// 512 bytes = 384 KiB per CTA (one CTA per SM), 8 rows in flight per warp,
// 8-deep look-back (256 predecessors per round trip), and warps 1..23 load
// and locally scan their first phase-3 rows while warp 0 looks back.
constexpr int L2_WARPS = 24, L2_ROWS = 32, L2_UNROLL = 8, L2_DEPTH = 8;
// Fallback for arrays that are not 16-byte aligned: register tile of
// 256 threads x 16 scalar-loaded items.
constexpr int RG_BLOCK = 256, RG_ITEMS = 16, RG_DEPTH = 4;

template <typename T>
constexpr int64_t l2_tile() {
  return (int64_t)L2_WARPS * L2_ROWS * 512 / (int64_t)sizeof(T);
}

template <typename T>
size_t ws_bytes(int64_t n) {
  // status for the smaller of the two tile sizes (either path may run)
  const int64_t min_tile = std::min<int64_t>(l2_tile<T>(), (int64_t)RG_BLOCK * RG_ITEMS);
  return HEADER + status_bytes<T>(cdiv(n, min_tile));
}

// Tin != T: the widened scans (int32 -> int64, float -> double; NEXT-2),
// same kernels, the input converted on load; a widened row stores 32 bytes
// per lane, so the super-tile path needs a 32-byte aligned output.
template <int OP, typename T, typename Tin, bool EXCLUSIVE>
ga_status_t run(int64_t n, const void *in, void *out, const void *carry, int64_t carry_count, void *ws,
                cudaStream_t s) {
  constexpr uintptr_t OUT_ALIGN = sizeof(T) == sizeof(Tin) ? 16 : 32;
  const bool aligned = ((uintptr_t)in & 15) == 0 && ((uintptr_t)out & (OUT_ALIGN - 1)) == 0;
  const bool inplace = in == out;
  if (aligned) {
    ScanArgs<T, Tin> p = make_args<T, Tin>(n, l2_tile<Tin>(), in, out, carry, carry_count, ws);
    const int grid = (int)p.num_tiles;
    if (inplace)
      scan_l2_kernel<OP, T, Tin, L2_WARPS, L2_ROWS, L2_UNROLL, L2_DEPTH, false, EXCLUSIVE, true>
          <<<grid, L2_WARPS * 32, 0, s>>>(p);
    else
      scan_l2_kernel<OP, T, Tin, L2_WARPS, L2_ROWS, L2_UNROLL, L2_DEPTH, true, EXCLUSIVE, true>
          <<<grid, L2_WARPS * 32, 0, s>>>(p);
  } else {
    ScanArgs<T, Tin> p = make_args<T, Tin>(n, (int64_t)RG_BLOCK * RG_ITEMS, in, out, carry, carry_count, ws);
    if (p.num_tiles > 0x7fffffffLL) return fail(GA_ERR_UNSUPPORTED, "scan: n too large (%lld)", (long long)n);
    scan_reg_kernel<OP, T, Tin, RG_BLOCK, RG_ITEMS, RG_DEPTH, EXCLUSIVE><<<(int)p.num_tiles, RG_BLOCK, 0, s>>>(p);
  }
  count_launch();
  return check_launch("scan_kernel");
}

template <int OP, typename T, typename Tin>
ga_status_t by_kind(bool ex, int64_t n, const void *in, void *out, const void *carry, int64_t cc, void *ws,
                    cudaStream_t s) {
  return ex ? run<OP, T, Tin, true>(n, in, out, carry, cc, ws, s)
            : run<OP, T, Tin, false>(n, in, out, carry, cc, ws, s);
}

template <typename T, typename Tin = T>
ga_status_t by_op(ga_op_t op, bool ex, int64_t n, const void *in, void *out, const void *carry, int64_t cc, void *ws,
                  cudaStream_t s) {
  switch (op) {
    case GA_OP_SUM: return by_kind<GA_OP_SUM, T, Tin>(ex, n, in, out, carry, cc, ws, s);
    case GA_OP_MAX: return by_kind<GA_OP_MAX, T, Tin>(ex, n, in, out, carry, cc, ws, s);
    case GA_OP_MIN: return by_kind<GA_OP_MIN, T, Tin>(ex, n, in, out, carry, cc, ws, s);
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad op %d", (int)op);
}

}  // namespace

size_t scan_workspace_bytes(ga_dtype_t dt, int64_t n) {
  switch (dt) {
    case GA_I32: return ws_bytes<int32_t>(n);
    case GA_I64: return ws_bytes<int64_t>(n);
    case GA_F32: return ws_bytes<float>(n);
    case GA_F64: return ws_bytes<double>(n);
    default: return 0;
  }
}

ga_status_t launch_scan(ga_op_t op, ga_scan_kind_t kind, ga_dtype_t in_dt, ga_dtype_t dt, int64_t n, const void *in,
                        void *out, const void *carry, int64_t carry_count, void *ws, cudaStream_t s) {
  const bool ex = kind == GA_SCAN_EXCLUSIVE;
  if (in_dt != dt) {
    if (in_dt == GA_I32 && dt == GA_I64) return by_op<int64_t, int32_t>(op, ex, n, in, out, carry, carry_count, ws, s);
    if (in_dt == GA_F32 && dt == GA_F64) return by_op<double, float>(op, ex, n, in, out, carry, carry_count, ws, s);
    return fail(GA_ERR_UNSUPPORTED, "scan %d -> %d not instantiated", (int)in_dt, (int)dt);
  }
  switch (dt) {
    case GA_I32: return by_op<int32_t>(op, ex, n, in, out, carry, carry_count, ws, s);
    case GA_I64: return by_op<int64_t>(op, ex, n, in, out, carry, carry_count, ws, s);
    case GA_F32: return by_op<float>(op, ex, n, in, out, carry, carry_count, ws, s);
    case GA_F64: return by_op<double>(op, ex, n, in, out, carry, carry_count, ws, s);
    default: break;
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad dtype %d", (int)dt);
}

}  // namespace ga
