// scan.cu — parallel prefix sum (§3.2.6: "GPU-based
// parallel prefix sums (also known as `parallel scan')") with the scan
// expressions "+", max, min (the reduction expressions of P:479-485) over
// int32 / int64 (wrapping, R4/R14) and float / double (R22).
//
// One launch, decoupled look-back across super-tiles (BASELINE.json
// north_star), HBM traffic 1 read + 1 write per element when the super-tiles
// in flight stay L2-resident (scan_l2_kernel in scan_kernel.cuh):
// The super-tile shape is chosen by size (scan_impl.cuh: smaller tiles for
// small n so every SM gets work); described here for the streaming shape L:
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
//     instruction (1 KiB rows — 32 bytes per lane — for the 8-byte and
//     widened scans when the arrays are 32-byte aligned);
//   - the ragged last tile has its own compiled body (vector accesses except
//     for the one lane straddling n).
// Look-back status words carry the call's epoch in every 64-bit word (for
// every element size, so one workspace may serve scans of any dtype, size and
// shape), so the workspace is zeroed once and never again (until the 30-bit
// epoch wraps: see gpuarray_scan_workspace_bytes); the CTA drawing the last
// id resets the counter.
// Tile 0's exclusive prefix is the carry-in c = sum(carry[0..carry_count)),
// which is how a sharded scan injects the totals of earlier shards.
// From 48 MiB of input up to 4 GiB (4-byte types), 2 GiB (8-byte) or
// without bound (widening) the single-touch ring scan runs instead
// (scan_ring.cuh: persistent CTAs, TMA stages, tiles held in registers while
// they look back, 4-byte tiles prefetched into L2 one draw ahead): 3-19%
// faster there; beyond, only the two-touch kernel's L2 buffer covers the
// look-back latency.
// The alternatives measured against this one (register-tiled single-touch,
// TMA-staged, warp-specialized, persistent look-ahead) are summarised in
// DESIGN.md §6, profiles/r1_scan_limits.md and profiles/r2_scan.md.
#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_impl.cuh"

namespace ga {
namespace scan_impl {
GA_SCAN_INSTANTIATE(SHAPE_RG)
}  // namespace scan_impl

using namespace scan_impl;

namespace {
template <typename T>
size_t ws_bytes(int64_t n) {
  // status for the smallest tile any path may use (the RG fallback's; every
  // super-tile shape has at least as many elements, also widened)
  static_assert(tile_elems<SHAPE_S, int32_t, int32_t>() >= tile_elems<SHAPE_RG, T, T>(), "RG tile is the smallest");
  static_assert(tile_elems<SHAPE_S, int64_t, int64_t>() >= tile_elems<SHAPE_RG, T, T>(), "RG tile is the smallest");
  return HEADER + status_bytes<T>(cdiv(n, tile_elems<SHAPE_RG, T, T>()));
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
  const size_t isz = dtype_size(in_dt), osz = dtype_size(dt);
  const uintptr_t out_align = isz == osz ? 16 : 32;
  const bool aligned = ((uintptr_t)in & 15) == 0 && ((uintptr_t)out & (out_align - 1)) == 0;
  if (!aligned) return launch_shape<SHAPE_RG>(op, ex, in_dt, dt, n, in, out, carry, carry_count, ws, s);
  if (use_ring(n, isz, osz, out)) return launch_ring(op, ex, in_dt, dt, n, in, out, carry, carry_count, ws, s);
  switch (choose_shape(n, isz, osz)) {
    case SHAPE_S: return launch_shape<SHAPE_S>(op, ex, in_dt, dt, n, in, out, carry, carry_count, ws, s);
    case SHAPE_M: return launch_shape<SHAPE_M>(op, ex, in_dt, dt, n, in, out, carry, carry_count, ws, s);
    default: return launch_shape<SHAPE_L>(op, ex, in_dt, dt, n, in, out, carry, carry_count, ws, s);
  }
}

}  // namespace ga
