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
// (red_detail::grid_finish), like reduce_kernel.  Arrays not 32-byte aligned
// take a scalar grid-stride loop (same arithmetic).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ga_device.cuh"
#include "ga_host.h"
#include "reduce_kernel.cuh"

namespace ga {
namespace {

using namespace red_detail;

constexpr int CG_BLOCK = 256, CG_UNROLL = 2, CG_MINB = 4;

template <typename T>
struct DirArgs {
  int64_t n, nvec;            // nvec = 0: scalar path for everything
  T bscale;                   // beta = RN(bscale * RN(*bnum / *bden))
  const T *bnum, *bden;
  T l, d, u;                  // operator tridiag(l, d_i, u)
  const T *diag;              // nullptr: constant d
  const T *r, *pin;
  T *pout, *ap;
  T *out, *partials;
  unsigned int *ticket;
};

template <typename T>
struct UpdArgs {
  int64_t n, nvec;
  T ascale;                   // alpha = RN(ascale * RN(*anum / *aden))
  const T *anum, *aden;
  T *x, *r;
  const T *p, *ap;
  T *out, *partials;
  unsigned int *ticket;
};

// p' = RN(RN(1*r) + RN(beta*p)) — gpuarray_axpbyz(1, r, beta, p) (R1).
template <typename T>
__device__ __forceinline__ T dir_p(T beta, T r, T p) {
  return e_add(e_mul(T(1), r), e_mul(beta, p));
}
template <typename T>
__device__ __forceinline__ T pnew_at(const DirArgs<T> &a, T beta, int64_t j) {
  return (j >= 0 && j < a.n) ? dir_p(beta, a.r[j], a.pin[j]) : T(0);
}
// (A p')_i with gpuarray_stencil3's operation order (R25).
template <typename T>
__device__ __forceinline__ T point(const DirArgs<T> &a, int64_t i, T pm, T p0, T pp, T di) {
  T acc = e_mul(di, p0);
  if (i > 0) acc = e_add(e_mul(a.l, pm), acc);
  if (i + 1 < a.n) acc = e_add(acc, e_mul(a.u, pp));
  return acc;
}

template <typename T, int VEC>
__device__ __forceinline__ T lane_tree(T (&acc)[VEC]) {
#pragma unroll
  for (int w = VEC / 2; w >= 1; w >>= 1) {
#pragma unroll
    for (int k = 0; k < w; ++k) acc[k] = e_add(acc[k], acc[k + w]);
  }
  return acc[0];
}

template <typename T>
__global__ void __launch_bounds__(CG_BLOCK, CG_MINB) cg_direction_kernel(DirArgs<T> a) {
  constexpr int VEC = 32 / sizeof(T);
  __shared__ T smem[CG_BLOCK / 32];
  const int lane = threadIdx.x & 31;
  const T beta = coef(a.bscale, a.bnum, a.bden);
  T acc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) acc[k] = T(0);

  // scalar part: everything after the last whole vector (or all of it)
  const int64_t tid = (int64_t)blockIdx.x * CG_BLOCK + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * CG_BLOCK;
  for (int64_t i = a.nvec * VEC + tid; i < a.n; i += nthreads) {
    const T p0 = pnew_at(a, beta, i);
    const T y = point(a, i, pnew_at(a, beta, i - 1), p0, pnew_at(a, beta, i + 1), a.diag ? a.diag[i] : a.d);
    a.pout[i] = p0;
    a.ap[i] = y;
    acc[VEC - 1] = e_fma(p0, y, acc[VEC - 1]);
  }

  constexpr int64_t CHUNK = (int64_t)CG_BLOCK * CG_UNROLL;
  for (int64_t base = (int64_t)blockIdx.x * CHUNK + threadIdx.x; base - threadIdx.x < a.nvec;
       base += (int64_t)gridDim.x * CHUNK) {
    V32 rv[CG_UNROLL], pv[CG_UNROLL], dv[CG_UNROLL];
    T hl[CG_UNROLL], hr[CG_UNROLL];  // halo p' (lane 0: left, lane 31 / last vector: right)
#pragma unroll
    for (int j = 0; j < CG_UNROLL; ++j) {
      const int64_t v = base + j * CG_BLOCK;
#pragma unroll
      for (int k = 0; k < 8; ++k) rv[j].r[k] = pv[j].r[k] = dv[j].r[k] = 0;
      hl[j] = hr[j] = T(0);
      if (v < a.nvec) {
        rv[j] = ld_nc_256(a.r + v * VEC);
        pv[j] = ld_nc_256(a.pin + v * VEC);
        if (a.diag) dv[j] = ld_nc_256(a.diag + v * VEC);
        if (lane == 0) hl[j] = pnew_at(a, beta, v * VEC - 1);
        if (lane == 31 || v + 1 >= a.nvec) hr[j] = pnew_at(a, beta, v * VEC + VEC);
      }
    }
#pragma unroll
    for (int j = 0; j < CG_UNROLL; ++j) {
      const int64_t v = base + j * CG_BLOCK;
      T pn[VEC];
#pragma unroll
      for (int k = 0; k < VEC; ++k) pn[k] = dir_p(beta, vget<T>(rv[j], k), vget<T>(pv[j], k));
      T left = __shfl_up_sync(0xffffffffu, pn[VEC - 1], 1);
      T right = __shfl_down_sync(0xffffffffu, pn[0], 1);
      if (v < a.nvec) {
        if (lane == 0) left = hl[j];
        if (lane == 31 || v + 1 >= a.nvec) right = hr[j];
        const int64_t i0 = v * VEC;
        V32 po, yo;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          const T di = a.diag ? vget<T>(dv[j], k) : a.d;
          const T y = point(a, i0 + k, k == 0 ? left : pn[k - 1], pn[k], k == VEC - 1 ? right : pn[k + 1], di);
          vset<T>(po, k, pn[k]);
          vset<T>(yo, k, y);
          acc[k] = e_fma(pn[k], y, acc[k]);
        }
        st_256(a.pout + i0, po);
        st_256(a.ap + i0, yo);
      }
    }
  }
  const T v = block_fold<GA_OP_SUM, CG_BLOCK, T>(lane_tree<T, VEC>(acc), smem);
  grid_finish<GA_OP_SUM, CG_BLOCK, T>(v, smem, a.partials, a.ticket, a.out, Exchange{});
}

template <typename T>
__global__ void __launch_bounds__(CG_BLOCK, CG_MINB) cg_update_kernel(UpdArgs<T> a) {
  constexpr int VEC = 32 / sizeof(T);
  __shared__ T smem[CG_BLOCK / 32];
  // x' = RN(RN(1*x) + RN(alpha*p)), r' = RN(RN(1*r) + RN(-alpha*ap)):
  // gpuarray_axpbyz_ds(1, x, alpha, p) and (1, r, -alpha, ap), whose b
  // factors are RN(+-ascale * q) = +-alpha exactly.
  const T alpha = coef(a.ascale, a.anum, a.aden);
  const T nalpha = coef(-a.ascale, a.anum, a.aden);
  T acc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) acc[k] = T(0);

  const int64_t tid = (int64_t)blockIdx.x * CG_BLOCK + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * CG_BLOCK;
  for (int64_t i = a.nvec * VEC + tid; i < a.n; i += nthreads) {
    a.x[i] = e_add(e_mul(T(1), a.x[i]), e_mul(alpha, a.p[i]));
    const T rn = e_add(e_mul(T(1), a.r[i]), e_mul(nalpha, a.ap[i]));
    a.r[i] = rn;
    acc[VEC - 1] = e_fma(rn, rn, acc[VEC - 1]);
  }

  constexpr int64_t CHUNK = (int64_t)CG_BLOCK * CG_UNROLL;
  for (int64_t base = (int64_t)blockIdx.x * CHUNK + threadIdx.x; base - threadIdx.x < a.nvec;
       base += (int64_t)gridDim.x * CHUNK) {
    V32 xv[CG_UNROLL], pv[CG_UNROLL], rv[CG_UNROLL], av[CG_UNROLL];
#pragma unroll
    for (int j = 0; j < CG_UNROLL; ++j) {
      const int64_t v = base + j * CG_BLOCK;
      if (v < a.nvec) {
        // x and r are rewritten in place: coherent loads
        xv[j] = ld_256(a.x + v * VEC);
        rv[j] = ld_256(a.r + v * VEC);
        pv[j] = ld_nc_256(a.p + v * VEC);
        av[j] = ld_nc_256(a.ap + v * VEC);
      }
    }
#pragma unroll
    for (int j = 0; j < CG_UNROLL; ++j) {
      const int64_t v = base + j * CG_BLOCK;
      if (v < a.nvec) {
        V32 xo, ro;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          vset<T>(xo, k, e_add(e_mul(T(1), vget<T>(xv[j], k)), e_mul(alpha, vget<T>(pv[j], k))));
          const T rn = e_add(e_mul(T(1), vget<T>(rv[j], k)), e_mul(nalpha, vget<T>(av[j], k)));
          vset<T>(ro, k, rn);
          acc[k] = e_fma(rn, rn, acc[k]);
        }
        st_256(a.x + v * VEC, xo);
        st_256(a.r + v * VEC, ro);
      }
    }
  }
  const T v = block_fold<GA_OP_SUM, CG_BLOCK, T>(lane_tree<T, VEC>(acc), smem);
  grid_finish<GA_OP_SUM, CG_BLOCK, T>(v, smem, a.partials, a.ticket, a.out, Exchange{});
}

template <typename T>
T sval(const ga_scalar_t &s);
template <>
float sval<float>(const ga_scalar_t &s) { return s.v.f32; }
template <>
double sval<double>(const ga_scalar_t &s) { return s.v.f64; }

bool aligned32(const void *p) { return ((uintptr_t)p & 31) == 0; }

// One CTA per CG_BLOCK * CG_UNROLL vectors (or CG_BLOCK scalars on the
// unaligned path), capped at RED_MAX_PARTIALS (chunks then repeat).
int grid_for(int64_t n, int64_t nvec) {
  const int64_t units = nvec > 0 ? cdiv(nvec, (int64_t)CG_BLOCK * CG_UNROLL) : cdiv(n, (int64_t)CG_BLOCK);
  return (int)std::max<int64_t>(std::min<int64_t>(units, RED_MAX_PARTIALS), 1);
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
  a.ticket = static_cast<unsigned int *>(ws);
  a.partials = reinterpret_cast<T *>(static_cast<char *>(ws) + RED_HEADER);
  const bool vec = aligned32(r) && aligned32(pin) && aligned32(pout) && aligned32(ap) && (!diag || aligned32(diag));
  a.nvec = vec ? n / VEC : 0;
  cg_direction_kernel<T><<<grid_for(n, a.nvec), CG_BLOCK, 0, s>>>(a);
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
  a.ticket = static_cast<unsigned int *>(ws);
  a.partials = reinterpret_cast<T *>(static_cast<char *>(ws) + RED_HEADER);
  const bool vec = aligned32(x) && aligned32(r) && aligned32(p) && aligned32(ap);
  a.nvec = vec ? n / VEC : 0;
  cg_update_kernel<T><<<grid_for(n, a.nvec), CG_BLOCK, 0, s>>>(a);
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
