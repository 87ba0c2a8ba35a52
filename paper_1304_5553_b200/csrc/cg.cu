// cg.cu — the two fused steps of one conjugate-gradient iteration, the
// second workload of SURVEY.md §8(f) NEXT-4 (the paper's "conjugate-gradient-
// based Krylov solver"), each ONE kernel that does what
// three hot-path calls would do, with the same per-element rounding:
//
//   gpuarray_cg_direction   p' = r + beta p         (axpbyz, a = 1, R1)
//                           ap = A p'               (stencil3, R25)
//                           pap = p' . ap           (dot, R9/R10)
//       HBM: read r, p; write p', ap = 4 element-sizes (16 B/elt fp32)
//       instead of 3 + 2 + 2 = 7 for the three calls;
//   gpuarray_cg_update      x' = x + alpha p        (axpbyz, a = 1)
//                           r' = r - alpha ap       (axpbyz, a = 1, b = -alpha)
//                           rr = r' . r'            (norm2sq)
//       HBM: read x, r, p, ap; write x', r' = 6 element-sizes instead of
//       3 + 3 + 1 = 7.
// One iteration = 2 launches and 10 element-sizes instead of 6 launches and
// 14.  beta and alpha are device-resident factors (ga_dscalar_t: the previous
// reductions' results stay on the GPU), so iterations can
// be captured in a CUDA graph with no host round trip.
//
// Layout: the one-shot grid of the reductions (CTA b owns CG_BLOCK * UNROLL
// consecutive 32-byte vectors; consecutive lanes hold consecutive vectors),
// so the stencil's neighbours come from warp shuffles and only lanes 0 / 31
// load one halo element each (computing p' there from r and p, the same
// bits).  The dot products accumulate per vector lane, fold in the fixed lane
// tree / warp butterfly / block order and finish in the last block
// (red_detail::grid_finish, tagged slots), like reduce_kernel.  Arrays not 32-byte aligned
// take a scalar grid-stride loop (same arithmetic).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "cg_kernel.cuh"

namespace ga {
namespace {

using namespace cg_detail;

// Tuned shape (tools/lab/run_cg_lab.py, profiles/r1_cg.md): one 32-byte
// vector per array per thread and pass, >= 4 CTAs per SM (64 registers), and
// each CTA making up to 4 passes (fewer CTAs => fewer block folds and
// finish slots): direction 6.1-6.3 TB/s, update 6.8 TB/s at 2^26 fp32.
constexpr int DIR_UNROLL = 1, DIR_MINB = 4, UPD_UNROLL = 1, UPD_MINB = 4, MAX_PASSES = 4;

template <typename T>
T sval(const ga_scalar_t &s);
template <>
float sval<float>(const ga_scalar_t &s) { return s.v.f32; }
template <>
double sval<double>(const ga_scalar_t &s) { return s.v.f64; }

bool aligned32(const void *p) { return ((uintptr_t)p & 31) == 0; }

// Grid: a chunk is CG_BLOCK * unroll vectors (CG_BLOCK scalars on the
// unaligned path); up to MAX_PASSES chunks per CTA as long as every SM still
// gets 4 CTAs; capped at RED_MAX_PARTIALS (chunks then repeat).
int grid_for(int64_t n, int64_t nvec, int unroll) {
  const int64_t chunks = nvec > 0 ? cdiv(nvec, (int64_t)CG_BLOCK * unroll) : cdiv(n, (int64_t)CG_BLOCK);
  const int64_t grid = std::max(cdiv(chunks, (int64_t)MAX_PASSES), std::min<int64_t>(chunks, 4LL * sm_count()));
  return (int)std::max<int64_t>(std::min<int64_t>(grid, RED_MAX_PARTIALS), 1);
}

template <typename T>
ga_status_t run_direction(int64_t n, const ga_dscalar_t &beta, const void *r, const void *pin, void *pout,
                          const ga_scalar_t &l, const ga_scalar_t &d, const ga_scalar_t &u, const void *diag,
                          void *ap, void *pap, void *ws, cudaStream_t s) {
  constexpr int VEC = 32 / sizeof(T);
  DirArgs<T> a;
  a.n = n;
  a.bscale = sval<T>(beta.scale);
  a.bnum = static_cast<const T *>(beta.num);
  a.bden = static_cast<const T *>(beta.den);
  a.l = sval<T>(l);
  a.d = sval<T>(d);
  a.u = sval<T>(u);
  a.diag = static_cast<const T *>(diag);
  a.r = static_cast<const T *>(r);
  a.pin = static_cast<const T *>(pin);
  a.pout = static_cast<T *>(pout);
  a.ap = static_cast<T *>(ap);
  a.out = static_cast<T *>(pap);
  const bool vec = aligned32(r) && aligned32(pin) && aligned32(pout) && aligned32(ap) && (!diag || aligned32(diag));
  a.nvec = vec ? n / VEC : 0;
  const int grid = grid_for(n, a.nvec, DIR_UNROLL);
  a.fin = make_finish(ws, grid, DIR_MINB);
  if (diag)
    launch(cg_direction_kernel<T, DIR_UNROLL, DIR_MINB, true>, grid, CG_BLOCK, 0, s, a);
  else
    launch(cg_direction_kernel<T, DIR_UNROLL, DIR_MINB, false>, grid, CG_BLOCK, 0, s, a);
  count_launch();
  return check_launch("cg_direction_kernel");
}

template <typename T>
ga_status_t run_update(int64_t n, const ga_dscalar_t &alpha, void *x, void *r, const void *p, const void *ap,
                       void *rr, void *ws, cudaStream_t s) {
  constexpr int VEC = 32 / sizeof(T);
  UpdArgs<T> a;
  a.n = n;
  a.ascale = sval<T>(alpha.scale);
  a.anum = static_cast<const T *>(alpha.num);
  a.aden = static_cast<const T *>(alpha.den);
  a.x = static_cast<T *>(x);
  a.r = static_cast<T *>(r);
  a.p = static_cast<const T *>(p);
  a.ap = static_cast<const T *>(ap);
  a.out = static_cast<T *>(rr);
  const bool vec = aligned32(x) && aligned32(r) && aligned32(p) && aligned32(ap);
  a.nvec = vec ? n / VEC : 0;
  const int grid = grid_for(n, a.nvec, UPD_UNROLL);
  a.fin = make_finish(ws, grid, UPD_MINB);
  launch(cg_update_kernel<T, UPD_UNROLL, UPD_MINB>, grid, CG_BLOCK, 0, s, a);
  count_launch();
  return check_launch("cg_update_kernel");
}

}  // namespace

ga_status_t launch_cg_direction(ga_dtype_t dt, int64_t n, const ga_dscalar_t &beta, const void *r, const void *pin,
                                void *pout, const ga_scalar_t &l, const ga_scalar_t &d, const ga_scalar_t &u,
                                const void *diag, void *ap, void *pap, void *ws, cudaStream_t s) {
  if (dt == GA_F32) return run_direction<float>(n, beta, r, pin, pout, l, d, u, diag, ap, pap, ws, s);
  return run_direction<double>(n, beta, r, pin, pout, l, d, u, diag, ap, pap, ws, s);
}

ga_status_t launch_cg_update(ga_dtype_t dt, int64_t n, const ga_dscalar_t &alpha, void *x, void *r, const void *p,
                             const void *ap, void *rr, void *ws, cudaStream_t s) {
  if (dt == GA_F32) return run_update<float>(n, alpha, x, r, p, ap, rr, ws, s);
  return run_update<double>(n, alpha, x, r, p, ap, rr, ws, s);
}

}  // namespace ga
