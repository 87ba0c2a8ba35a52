// stencil.cu — three-point stencil / tridiagonal matvec, the operator of the
// CG workload (§8(f) NEXT-4: the paper's "conjugate-gradient-based Krylov
// solver", applied matrix-free to 1-D Poisson-type
// systems):  y_i = l*x_{i-1} + d_i*x_i + u*x_{i+1}, boundary terms omitted,
// each operation RN left to right (R25):
//   y_i = RN(RN(RN(l*x_{i-1}) + RN(d_i*x_i)) + RN(u*x_{i+1})).
// HBM-bound: 8 B/elt fp32 (read x, write y; +4 B with a diagonal array).
// One-shot grid of 256-bit vectors; the neighbours across vector boundaries
// come from warp shuffles, across warp boundaries from (cached) scalar loads.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ga_device.cuh"
#include "ga_host.h"

namespace ga {
namespace {

constexpr int ST_BLOCK = 256;

template <typename T>
struct StArgs {
  int64_t n;
  int64_t nvec;  // whole 32-byte vectors (the remainder is the scalar tail)
  T l, d, u;
  const T *diag;  // nullptr: constant d
  const T *x;
  T *y;
};

template <typename T>
__device__ __forceinline__ T point(const StArgs<T> &p, int64_t i, T xm, T x0, T xp) {
  const T di = p.diag ? p.diag[i] : p.d;
  T acc = e_mul(di, x0);
  if (i > 0) acc = e_add(e_mul(p.l, xm), acc);
  if (i + 1 < p.n) acc = e_add(acc, e_mul(p.u, xp));
  return acc;
}

template <typename T>
__global__ void __launch_bounds__(ST_BLOCK) stencil_vec_kernel(StArgs<T> p) {
  pdl_enter();
  constexpr int VEC = 32 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t v = (int64_t)blockIdx.x * ST_BLOCK + threadIdx.x;
  // scalar tail after the last whole vector
  const int64_t tail0 = p.nvec * VEC;
  if (v < p.n - tail0) {
    const int64_t i = tail0 + v;
    p.y[i] = point(p, i, i > 0 ? p.x[i - 1] : T(0), p.x[i], i + 1 < p.n ? p.x[i + 1] : T(0));
  }
  const bool live = v < p.nvec;
  V32 xv;
#pragma unroll
  for (int k = 0; k < 8; ++k) xv.r[k] = 0;
  if (live) xv = ld_nc_256(p.x + v * VEC);
  // neighbours of the vector's first / last element
  T left = __shfl_up_sync(0xffffffffu, vget<T>(xv, VEC - 1), 1);
  T right = __shfl_down_sync(0xffffffffu, vget<T>(xv, 0), 1);
  if (!live) return;
  const int64_t i0 = v * VEC;
  if (lane == 0 || v == (int64_t)blockIdx.x * ST_BLOCK) left = i0 > 0 ? p.x[i0 - 1] : T(0);
  if (lane == 31 || v + 1 >= p.nvec) right = i0 + VEC < p.n ? p.x[i0 + VEC] : T(0);
  V32 yv;
#pragma unroll
  for (int k = 0; k < VEC; ++k) {
    const T xm = k == 0 ? left : vget<T>(xv, k - 1);
    const T xp = k == VEC - 1 ? right : vget<T>(xv, k + 1);
    vset<T>(yv, k, point(p, i0 + k, xm, vget<T>(xv, k), xp));
  }
  st_256(p.y + i0, yv);
}

template <typename T>
__global__ void __launch_bounds__(ST_BLOCK) stencil_scalar_kernel(StArgs<T> p) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * ST_BLOCK;
  for (int64_t i = (int64_t)blockIdx.x * ST_BLOCK + threadIdx.x; i < p.n; i += stride)
    p.y[i] = point(p, i, i > 0 ? p.x[i - 1] : T(0), p.x[i], i + 1 < p.n ? p.x[i + 1] : T(0));
}

template <typename T>
T sval(const ga_scalar_t &s);
template <>
float sval<float>(const ga_scalar_t &s) { return s.v.f32; }
template <>
double sval<double>(const ga_scalar_t &s) { return s.v.f64; }

template <typename T>
ga_status_t run(int64_t n, const ga_scalar_t &l, const ga_scalar_t &d, const ga_scalar_t &u, const void *diag,
                const void *x, void *y, cudaStream_t s) {
  constexpr int VEC = 32 / sizeof(T);
  StArgs<T> p;
  p.n = n;
  p.l = sval<T>(l);
  p.d = sval<T>(d);
  p.u = sval<T>(u);
  p.diag = static_cast<const T *>(diag);
  p.x = static_cast<const T *>(x);
  p.y = static_cast<T *>(y);
  const bool aligned = ((uintptr_t)x & 31) == 0 && ((uintptr_t)y & 31) == 0;
  if (aligned) {
    p.nvec = n / VEC;
    const int64_t threads = std::max<int64_t>(p.nvec, n - p.nvec * VEC);
    const int grid = (int)std::max<int64_t>(cdiv(threads, ST_BLOCK), 1);
    launch(stencil_vec_kernel<T>, grid, ST_BLOCK, 0, s, p);
  } else {
    p.nvec = 0;
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(cdiv(n, ST_BLOCK), 1), (int64_t)sm_count() * 16);
    launch(stencil_scalar_kernel<T>, grid, ST_BLOCK, 0, s, p);
  }
  count_launch();
  return check_launch("stencil_kernel");
}

}  // namespace

ga_status_t launch_stencil3(ga_dtype_t dt, int64_t n, const ga_scalar_t &l, const ga_scalar_t &d,
                            const ga_scalar_t &u, const void *diag, const void *x, void *y, cudaStream_t s) {
  if (dt == GA_F32) return run<float>(n, l, d, u, diag, x, y, s);
  if (dt == GA_F64) return run<double>(n, l, d, u, diag, x, y, s);
  return fail(GA_ERR_UNSUPPORTED, "stencil3: dtype %d not instantiated (F32, F64)", (int)dt);
}

}  // namespace ga
