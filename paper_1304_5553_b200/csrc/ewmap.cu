// ewmap.cu — GPUArray's other arithmetic operators and cumath-style unary
// maps (§8(f) NEXT-2; "They support all arithmetic operators ... many
// special functions are available in pycuda.cumath"):
//   binary z = x*y, x/y, maxNum(x,y), minNum(x,y); unary sqrt, |x|, -x,
//   exp, log, sin, cos.
// IEEE-exact operations use the _rn intrinsics (bit-exact against the
// oracle); exp/log/sin/cos use CUDA's accurate (non-fast-math) device
// functions, within DESIGN.md R26's ulp bound of glibc.  Integers: x*y
// (wrapping), |x|, -x (wrapping at INT_MIN), max, min.
// HBM-bound: 12 B/elt binary, 8 B/elt unary (fp32).  Same one-shot 256-bit
// vector structure as elementwise.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ga_device.cuh"
#include "ga_host.h"

namespace ga {
namespace {

constexpr int EM_BLOCK = 512;

template <int OP>
constexpr bool binary_op() {
  return OP == GA_EW_MUL || OP == GA_EW_DIV || OP == GA_EW_MAX || OP == GA_EW_MIN;
}

template <int OP, typename T>
__device__ __forceinline__ T apply(T a, T b) {
  if constexpr (std::is_floating_point<T>::value) {
    constexpr bool F = std::is_same<T, float>::value;
    if constexpr (OP == GA_EW_MUL) return e_mul(a, b);
    else if constexpr (OP == GA_EW_DIV) return e_div(a, b);
    else if constexpr (OP == GA_EW_SQRT) { if constexpr (F) return __fsqrt_rn(a); else return __dsqrt_rn(a); }
    else if constexpr (OP == GA_EW_ABS) return F ? fabsf(a) : fabs(a);
    else if constexpr (OP == GA_EW_NEG) return -a;
    else if constexpr (OP == GA_EW_EXP) { if constexpr (F) return expf(a); else return exp(a); }
    else if constexpr (OP == GA_EW_LOG) { if constexpr (F) return logf(a); else return log(a); }
    else if constexpr (OP == GA_EW_SIN) { if constexpr (F) return sinf(a); else return sin(a); }
    else if constexpr (OP == GA_EW_COS) { if constexpr (F) return cosf(a); else return cos(a); }
    else if constexpr (OP == GA_EW_MAX) return Op<GA_OP_MAX, T>::fold(a, b);
    else return Op<GA_OP_MIN, T>::fold(a, b);
  } else {
    using U = typename std::make_unsigned<T>::type;
    if constexpr (OP == GA_EW_MUL) return e_mul(a, b);
    else if constexpr (OP == GA_EW_ABS) return a < 0 ? (T)(U(0) - (U)a) : a;
    else if constexpr (OP == GA_EW_NEG) return (T)(U(0) - (U)a);
    else if constexpr (OP == GA_EW_MAX) return a > b ? a : b;
    else return a < b ? a : b;  // GA_EW_MIN
  }
}

template <typename T>
struct EmArgs {
  int64_t n, head, nvec;
  const T *x;
  const T *y;
  T *z;
};

template <int OP, typename T, int UNROLL, bool NC>
__global__ void __launch_bounds__(EM_BLOCK) ewmap_vec_kernel(EmArgs<T> p) {
  pdl_enter();
  constexpr int VEC = 32 / sizeof(T);
  constexpr bool HAS_Y = binary_op<OP>();
  const int64_t tid = (int64_t)blockIdx.x * EM_BLOCK + threadIdx.x;
  const int64_t tail0 = p.head + p.nvec * VEC;
  if (tid < p.head) p.z[tid] = apply<OP, T>(p.x[tid], HAS_Y ? p.y[tid] : T(0));
  if (tid < p.n - tail0) p.z[tail0 + tid] = apply<OP, T>(p.x[tail0 + tid], HAS_Y ? p.y[tail0 + tid] : T(0));
  const char *xb = reinterpret_cast<const char *>(p.x + p.head);
  const char *yb = HAS_Y ? reinterpret_cast<const char *>(p.y + p.head) : nullptr;
  char *zb = reinterpret_cast<char *>(p.z + p.head);
  constexpr int64_t CHUNK = (int64_t)EM_BLOCK * UNROLL;
  for (int64_t base = (int64_t)blockIdx.x * CHUNK + threadIdx.x; base < p.nvec; base += (int64_t)gridDim.x * CHUNK) {
    V32 vx[UNROLL], vy[UNROLL];
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      const int64_t v = base + j * EM_BLOCK;
      if (v < p.nvec) {
        vx[j] = ld_vec<NC>(xb + v * 32);
        if constexpr (HAS_Y) vy[j] = ld_vec<NC>(yb + v * 32);
      }
    }
#pragma unroll
    for (int j = 0; j < UNROLL; ++j) {
      const int64_t v = base + j * EM_BLOCK;
      if (v < p.nvec) {
        V32 vz;
#pragma unroll
        for (int k = 0; k < VEC; ++k)
          vset<T>(vz, k, apply<OP, T>(vget<T>(vx[j], k), HAS_Y ? vget<T>(vy[j], k) : T(0)));
        st_256(zb + v * 32, vz);
      }
    }
  }
}

template <int OP, typename T>
__global__ void __launch_bounds__(EM_BLOCK) ewmap_scalar_kernel(EmArgs<T> p) {
  pdl_enter();
  constexpr bool HAS_Y = binary_op<OP>();
  const int64_t stride = (int64_t)gridDim.x * EM_BLOCK;
  for (int64_t i = (int64_t)blockIdx.x * EM_BLOCK + threadIdx.x; i < p.n; i += stride)
    p.z[i] = apply<OP, T>(p.x[i], HAS_Y ? p.y[i] : T(0));
}

template <int OP, typename T>
ga_status_t run(int64_t n, const void *x, const void *y, void *z, cudaStream_t s) {
  constexpr int VEC = 32 / sizeof(T);
  constexpr bool HAS_Y = binary_op<OP>();
  constexpr int UNROLL = HAS_Y ? 2 : 4;
  EmArgs<T> p;
  p.n = n;
  p.x = static_cast<const T *>(x);
  p.y = static_cast<const T *>(y);
  p.z = static_cast<T *>(z);
  const uintptr_t phase = (uintptr_t)x & 31;
  const bool coaligned = ((uintptr_t)z & 31) == phase && (!HAS_Y || ((uintptr_t)y & 31) == phase) &&
                         (phase % sizeof(T)) == 0;
  if (!coaligned) {
    p.head = p.nvec = 0;
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(cdiv(n, EM_BLOCK), 1), (int64_t)sm_count() * 8);
    launch(ewmap_scalar_kernel<OP, T>, grid, EM_BLOCK, 0, s, p);
  } else {
    p.head = std::min<int64_t>(n, (int64_t)(((32 - phase) & 31) / sizeof(T)));
    p.nvec = (n - p.head) / VEC;
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(cdiv(p.nvec, (int64_t)EM_BLOCK * UNROLL), 1),
                                            0x7fffffffLL);
    const bool inplace = z == x || (HAS_Y && z == y);
    if (inplace) launch(ewmap_vec_kernel<OP, T, UNROLL, false>, grid, EM_BLOCK, 0, s, p);
    else launch(ewmap_vec_kernel<OP, T, UNROLL, true>, grid, EM_BLOCK, 0, s, p);
  }
  count_launch();
  return check_launch("ewmap_kernel");
}

template <typename T>
ga_status_t by_op(ga_ewop_t op, int64_t n, const void *x, const void *y, void *z, cudaStream_t s) {
  constexpr bool FP = std::is_floating_point<T>::value;
  switch (op) {
    case GA_EW_MUL: return run<GA_EW_MUL, T>(n, x, y, z, s);
    case GA_EW_ABS: return run<GA_EW_ABS, T>(n, x, y, z, s);
    case GA_EW_NEG: return run<GA_EW_NEG, T>(n, x, y, z, s);
    case GA_EW_MAX: return run<GA_EW_MAX, T>(n, x, y, z, s);
    case GA_EW_MIN: return run<GA_EW_MIN, T>(n, x, y, z, s);
    default: break;
  }
  if constexpr (FP) {
    switch (op) {
      case GA_EW_DIV: return run<GA_EW_DIV, T>(n, x, y, z, s);
      case GA_EW_SQRT: return run<GA_EW_SQRT, T>(n, x, y, z, s);
      case GA_EW_EXP: return run<GA_EW_EXP, T>(n, x, y, z, s);
      case GA_EW_LOG: return run<GA_EW_LOG, T>(n, x, y, z, s);
      case GA_EW_SIN: return run<GA_EW_SIN, T>(n, x, y, z, s);
      case GA_EW_COS: return run<GA_EW_COS, T>(n, x, y, z, s);
      default: break;
    }
  }
  return fail(GA_ERR_UNSUPPORTED, "elementwise op %d not instantiated for this dtype", (int)op);
}

}  // namespace

bool ewop_binary(ga_ewop_t op) { return op == GA_EW_MUL || op == GA_EW_DIV || op == GA_EW_MAX || op == GA_EW_MIN; }

ga_status_t launch_ewmap(ga_ewop_t op, ga_dtype_t dt, int64_t n, const void *x, const void *y, void *z,
                         cudaStream_t s) {
  switch (dt) {
    case GA_F32: return by_op<float>(op, n, x, y, z, s);
    case GA_F64: return by_op<double>(op, n, x, y, z, s);
    case GA_I32: return by_op<int32_t>(op, n, x, y, z, s);
    case GA_I64: return by_op<int64_t>(op, n, x, y, z, s);
    default: return fail(GA_ERR_UNSUPPORTED, "elementwise: dtype %d not instantiated", (int)dt);
  }
}

}  // namespace ga
