// elementwise.cu — ElementwiseKernel-style fused linear combinations
// (§3.2.4): "a statement ... to be executed for each value
// of i", evaluated "in a single pass" so no temporaries
// are created.
//
//   axpbyz: z[i] = a*x[i] + b*y[i]     12 B/elt fp32 (read x, y; write z)
//   axpbz : z[i] = a*x[i] + b           8 B/elt fp32
//
// HBM-bound (0.25 flop/B).  B200 design: a one-shot grid (no grid-stride
// wave) where CTA b owns the contiguous chunk of EW_BLOCK*UNROLL 32-byte
// vectors starting at b*EW_BLOCK*UNROLL; 256-bit vector loads/stores
// (LDG/STG.256, one 1 KiB contiguous request per warp instruction), all
// UNROLL vectors of a thread loaded before any is used, L1 bypassed (data is
// touched once).  tools/lab/ew_lab.cu measured this shape at 7.0 TB/s against
// 6.3-6.5 TB/s for a persistent grid-stride wave (n = 2^28 fp32).  A scalar
// head peels x/y/z to 32-byte alignment and a scalar tail finishes the
// remainder; arrays whose addresses differ modulo 32 B take a scalar path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ga_device.cuh"
#include "ga_host.h"

namespace ga {
namespace {

constexpr int EW_BLOCK = 512;

template <typename T>
struct EwArgs {
  int64_t n;     // elements
  int64_t head;  // scalar elements before the 32-byte aligned body
  int64_t nvec;  // 32-byte vectors in the body
  T a, b;
  const T *x;
  const T *y;  // unused by axpbz
  T *z;
  // device-resident scalar factors (gpuarray_axpbyz_ds): a = RN(a * RN(an / ad)),
  // a missing pointer standing for 1; all NULL: a and b as given
  const T *an = nullptr, *ad = nullptr, *bn = nullptr, *bd = nullptr;
};

// One element of the statement; the rounding sequence is DESIGN.md R1.
template <typename T, bool HAS_Y>
__device__ __forceinline__ T stmt(T a, T x, T b, T y) {
  if constexpr (HAS_Y) return e_add(e_mul(a, x), e_mul(b, y));
  else return e_add(e_mul(a, x), b);
}

// DS: the coefficients carry device-resident factors (gpuarray_axpbyz_ds);
// kept out of the plain instantiations, whose SASS must show only the R1
// sequence (the IEEE division behind the factors is itself FMA-based).
template <typename T, bool HAS_Y, int UNROLL, bool NC, bool DS>
__global__ void __launch_bounds__(EW_BLOCK) ew_vec_kernel(EwArgs<T> p) {
  pdl_enter();
  constexpr int VEC = 32 / sizeof(T);
  const int64_t tid = (int64_t)blockIdx.x * EW_BLOCK + threadIdx.x;
  if constexpr (DS) {
    p.a = coef(p.a, p.an, p.ad);
    p.b = coef(p.b, p.bn, p.bd);
  }

  // Scalar head (to 32 B alignment) and tail (remainder of the body).
  const int64_t tail0 = p.head + p.nvec * VEC;
  if (tid < p.head) {
    T y = HAS_Y ? p.y[tid] : zero_of<T>();
    p.z[tid] = stmt<T, HAS_Y>(p.a, p.x[tid], p.b, y);
  }
  if (tid < p.n - tail0) {
    int64_t i = tail0 + tid;
    T y = HAS_Y ? p.y[i] : zero_of<T>();
    p.z[i] = stmt<T, HAS_Y>(p.a, p.x[i], p.b, y);
  }

  const char *xb = reinterpret_cast<const char *>(p.x + p.head);
  const char *yb = HAS_Y ? reinterpret_cast<const char *>(p.y + p.head) : nullptr;
  char *zb = reinterpret_cast<char *>(p.z + p.head);

  // CTA b owns vectors [b*CHUNK, (b+1)*CHUNK), CHUNK = EW_BLOCK*UNROLL; the
  // loop only repeats if the grid was capped (n beyond 2^31 CTAs' worth).
  constexpr int64_t CHUNK = (int64_t)EW_BLOCK * UNROLL;
  for (int64_t base = (int64_t)blockIdx.x * CHUNK + threadIdx.x; base < p.nvec; base += (int64_t)gridDim.x * CHUNK) {
    V32 vx[UNROLL], vy[UNROLL];
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      int64_t v = base + j * EW_BLOCK;
      if (v < p.nvec) {
        vx[j] = ld_vec<NC>(xb + v * 32);
        if constexpr (HAS_Y) vy[j] = ld_vec<NC>(yb + v * 32);
      }
    }
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      int64_t v = base + j * EW_BLOCK;
      if (v < p.nvec) {
        V32 vz;
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          T y = HAS_Y ? vget<T>(vy[j], k) : zero_of<T>();
          vset<T>(vz, k, stmt<T, HAS_Y>(p.a, vget<T>(vx[j], k), p.b, y));
        }
        st_256(zb + v * 32, vz);
      }
    }
  }
}

// Arrays not co-aligned modulo 32 B: scalar grid-stride loop, still one pass.
template <typename T, bool HAS_Y, bool DS>
__global__ void __launch_bounds__(EW_BLOCK) ew_scalar_kernel(EwArgs<T> p) {
  pdl_enter();
  const int64_t nthreads = (int64_t)gridDim.x * EW_BLOCK;
  if constexpr (DS) {
    p.a = coef(p.a, p.an, p.ad);
    p.b = coef(p.b, p.bn, p.bd);
  }
  for (int64_t i = (int64_t)blockIdx.x * EW_BLOCK + threadIdx.x; i < p.n; i += nthreads) {
    T y = HAS_Y ? p.y[i] : zero_of<T>();
    p.z[i] = stmt<T, HAS_Y>(p.a, p.x[i], p.b, y);
  }
}

template <typename T>
T scalar_value(const ga_scalar_t &s);
template <>
float scalar_value<float>(const ga_scalar_t &s) { return s.v.f32; }
template <>
double scalar_value<double>(const ga_scalar_t &s) { return s.v.f64; }
template <>
int32_t scalar_value<int32_t>(const ga_scalar_t &s) { return s.v.i32; }
template <>
int64_t scalar_value<int64_t>(const ga_scalar_t &s) { return s.v.i64; }
template <>
c64 scalar_value<c64>(const ga_scalar_t &s) { return c64{s.v.c64[0], s.v.c64[1]}; }
template <>
c128 scalar_value<c128>(const ga_scalar_t &s) { return c128{s.v.c128[0], s.v.c128[1]}; }

template <typename T, bool HAS_Y>
ga_status_t launch_ew(int64_t n, const ga_scalar_t &a, const void *x, const ga_scalar_t &b, const void *y,
                      void *z, cudaStream_t s, const void *an = nullptr, const void *ad = nullptr,
                      const void *bn = nullptr, const void *bd = nullptr) {
  constexpr int VEC = 32 / sizeof(T);
  constexpr int UNROLL = HAS_Y ? 2 : 4;
  constexpr int64_t CHUNK = (int64_t)EW_BLOCK * UNROLL;
  EwArgs<T> p;
  p.n = n;
  p.a = scalar_value<T>(a);
  p.b = scalar_value<T>(b);
  p.x = static_cast<const T *>(x);
  p.y = static_cast<const T *>(y);
  p.z = static_cast<T *>(z);
  p.an = static_cast<const T *>(an);
  p.ad = static_cast<const T *>(ad);
  p.bn = static_cast<const T *>(bn);
  p.bd = static_cast<const T *>(bd);
  const bool ds = an || ad || bn || bd;

  const uintptr_t phase = (uintptr_t)x & 31;
  const bool coaligned = ((uintptr_t)z & 31) == phase && (!HAS_Y || ((uintptr_t)y & 31) == phase) &&
                         (phase % sizeof(T)) == 0;
  if (!coaligned) {
    const int max_grid = resident_grid((const void *)ew_scalar_kernel<T, HAS_Y, false>, EW_BLOCK);
    int grid = (int)std::min<int64_t>(cdiv(n, EW_BLOCK), max_grid);
    p.head = 0;
    p.nvec = 0;
    if (ds) launch(ew_scalar_kernel<T, HAS_Y, true>, grid, EW_BLOCK, 0, s, p);
    else launch(ew_scalar_kernel<T, HAS_Y, false>, grid, EW_BLOCK, 0, s, p);
    count_launch();
    return check_launch("ew_scalar_kernel");
  }
  p.head = std::min<int64_t>(n, (int64_t)(((32 - phase) & 31) / sizeof(T)));
  p.nvec = (n - p.head) / VEC;
  // In-place (z == x or z == y) must use coherent loads: the .nc path
  // requires the data to stay unwritten for the kernel's lifetime.
  const bool inplace = z == x || (HAS_Y && z == y);
  int grid = (int)std::min<int64_t>(std::max<int64_t>(cdiv(p.nvec, CHUNK), 1), 0x7fffffffLL);
  if (ds) {
    if (inplace) launch(ew_vec_kernel<T, HAS_Y, UNROLL, false, true>, grid, EW_BLOCK, 0, s, p);
    else launch(ew_vec_kernel<T, HAS_Y, UNROLL, true, true>, grid, EW_BLOCK, 0, s, p);
  } else {
    if (inplace) launch(ew_vec_kernel<T, HAS_Y, UNROLL, false, false>, grid, EW_BLOCK, 0, s, p);
    else launch(ew_vec_kernel<T, HAS_Y, UNROLL, true, false>, grid, EW_BLOCK, 0, s, p);
  }
  count_launch();
  return check_launch("ew_vec_kernel");
}

}  // namespace

ga_status_t launch_axpbyz(ga_dtype_t dt, int64_t n, const ga_scalar_t &a, const void *x, const ga_scalar_t &b,
                          const void *y, void *z, cudaStream_t s) {
  switch (dt) {
    case GA_F32: return launch_ew<float, true>(n, a, x, b, y, z, s);
    case GA_F64: return launch_ew<double, true>(n, a, x, b, y, z, s);
    case GA_I32: return launch_ew<int32_t, true>(n, a, x, b, y, z, s);
    case GA_I64: return launch_ew<int64_t, true>(n, a, x, b, y, z, s);
    case GA_C64: return launch_ew<c64, true>(n, a, x, b, y, z, s);
    case GA_C128: return launch_ew<c128, true>(n, a, x, b, y, z, s);
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "bad dtype %d", (int)dt);
}

ga_status_t launch_axpbyz_ds(ga_dtype_t dt, int64_t n, const ga_scalar_t &a, const void *an, const void *ad,
                             const void *x, const ga_scalar_t &b, const void *bn, const void *bd, const void *y,
                             void *z, cudaStream_t s) {
  if (dt == GA_F32) return launch_ew<float, true>(n, a, x, b, y, z, s, an, ad, bn, bd);
  if (dt == GA_F64) return launch_ew<double, true>(n, a, x, b, y, z, s, an, ad, bn, bd);
  return fail(GA_ERR_UNSUPPORTED, "axpbyz_ds: device-scalar factors need F32 or F64");
}

ga_status_t launch_axpbz(ga_dtype_t dt, int64_t n, const ga_scalar_t &a, const void *x, const ga_scalar_t &b,
                         void *z, cudaStream_t s) {
  switch (dt) {
    case GA_F32: return launch_ew<float, false>(n, a, x, b, nullptr, z, s);
    case GA_F64: return launch_ew<double, false>(n, a, x, b, nullptr, z, s);
    case GA_I32: return launch_ew<int32_t, false>(n, a, x, b, nullptr, z, s);
    case GA_I64: return launch_ew<int64_t, false>(n, a, x, b, nullptr, z, s);
    case GA_C64: return launch_ew<c64, false>(n, a, x, b, nullptr, z, s);
    case GA_C128: return launch_ew<c128, false>(n, a, x, b, nullptr, z, s);
  }
  return fail(GA_ERR_INVALID_ARGUMENT, "bad dtype %d", (int)dt);
}

}  // namespace ga
