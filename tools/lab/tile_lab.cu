// tile_lab.cu — the PRODUCT scan_l2_kernel (scan_kernel.cuh) at other
// super-tile shapes, to choose the shape by n (small n: more, smaller tiles).
#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_kernel.cuh"

using namespace ga::scan_detail;

// PF: rows per warp prefetched into L2 for the tile PF_DIST ids ahead.
template <typename T, int W, int R, int U, int D, int P1U = U, int PF = 0, int PF_DIST = 148>
static int run(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int64_t TILE = (int64_t)W * R * 512 / sizeof(T);
  ScanArgs<T> p = make_args<T>(n, TILE, in, out, nullptr, 0, ws);
  p.pf_dist = PF_DIST;
  scan_l2_kernel<GA_OP_SUM, T, T, W, R, U, D, true, true, true, P1U, PF><<<(int)p.num_tiles, W * 32, 0, s>>>(p, nullptr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

#define V(X)                        \
  X(0, int32_t, 24, 32, 8, 8, 8)    \
  X(1, int32_t, 24, 32, 8, 8, 16)   \
  X(2, int32_t, 24, 32, 8, 8, 32)   \
  X(3, int32_t, 24, 32, 4, 8, 16)   \
  X(4, int32_t, 16, 32, 8, 8, 16)   \
  X(5, int32_t, 32, 16, 8, 8, 16)   \
  X(6, int32_t, 24, 64, 8, 8, 16)   \
  X(20, int64_t, 24, 32, 8, 4, 8)   \
  X(21, int64_t, 24, 32, 8, 4, 16)   \
  X(10, int32_t, 12, 32, 8, 8, 8)   \
  X(11, int32_t, 12, 64, 8, 8, 8)   \
  X(12, int32_t, 8, 32, 8, 8, 8)    \
  X(13, int32_t, 8, 48, 8, 8, 8)    \
  X(14, int32_t, 12, 48, 8, 8, 8)   \
  X(15, int32_t, 8, 64, 8, 8, 8)    \
  X(16, int32_t, 12, 16, 8, 8, 8)   \
  X(22, int64_t, 12, 32, 8, 4, 8)   \
  X(23, int64_t, 12, 64, 8, 4, 8)   \
  X(24, int64_t, 8, 32, 8, 4, 8)    \
  X(7, int32_t, 32, 8, 8, 8, 8)     \
  X(8, int32_t, 8, 8, 8, 8, 8)      \
  X(9, int32_t, 8, 16, 8, 8, 8)     \
  X(25, int64_t, 32, 8, 4, 4, 8)    \
  X(26, int64_t, 16, 8, 4, 4, 8)    \
  X(27, int64_t, 12, 32, 4, 4, 8)   \
  X(28, int64_t, 8, 48, 4, 4, 8)    \
  X(29, int64_t, 8, 32, 4, 4, 8)

// prefetch variants: id, T, warps, rows, PF rows, distance, phase-3 rows (UNROLL), look-back depth, phase-1 rows (P1U)
#define PFV(X)                                  \
  X(40, int32_t, 24, 32, 32, 42, 8, 8, 8)         \
  X(41, int32_t, 24, 32, 32, 42, 8, 8, 16)        \
  X(42, int32_t, 24, 32, 32, 42, 8, 8, 4)         \
  X(43, int32_t, 24, 32, 32, 42, 4, 8, 8)         \
  X(44, int32_t, 24, 32, 32, 42, 8, 4, 8)         \
  X(45, int32_t, 24, 32, 32, 42, 8, 16, 8)        \
  X(47, int32_t, 24, 32, 32, 42, 16, 8, 16)       \
  X(46, int64_t, 24, 32, 32, 42, 4, 4, 8)         \
  X(50, int64_t, 24, 32, 32, 42, 4, 4, 16)        \
  X(51, int64_t, 24, 32, 32, 42, 4, 8, 8)         \
  X(170, int32_t, 24, 32, 32, 21, 8, 8, 8)         \
  X(171, int32_t, 24, 32, 32, 84, 8, 8, 8)         \
  X(172, int32_t, 24, 32, 32, 148, 8, 8, 8)        \
  X(173, int32_t, 24, 32, 32, 296, 8, 8, 8)       \
  X(174, int32_t, 24, 32, 32, 32, 8, 8, 8)        \
  X(175, int32_t, 24, 32, 32, 37, 8, 8, 8)        \
  X(176, int32_t, 24, 32, 32, 48, 8, 8, 8)        \
  X(177, int32_t, 24, 32, 32, 56, 8, 8, 8)

// 1 KiB rows (RB = 1024: LDG/STG.256): T, warps, rows, UNROLL, P1U, PF rows, distance
template <typename T, int W, int R, int U, int P1, int PF, int DIST, bool EX = true>
static int run_rb(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int64_t TILE = (int64_t)W * R * 1024 / sizeof(T);
  constexpr int D = sizeof(T) == 8 ? 4 : 8;
  ScanArgs<T> p = make_args<T>(n, TILE, in, out, nullptr, 0, ws);
  p.pf_dist = DIST;
  scan_l2_kernel<GA_OP_SUM, T, T, W, R, U, D, true, EX, true, P1, PF, false, 1024>
      <<<(int)p.num_tiles, W * 32, 0, s>>>(p, nullptr);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// widened int32 -> int64 with RB = 512 (product shape) or 1024
template <int RB, int R, int U, int P1>
static int run_wide(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int64_t TILE = 24 * 32 * 512 / 4;
  ScanArgs<int64_t, int32_t> p = make_args<int64_t, int32_t>(n, TILE, in, out, nullptr, 0, ws);
  scan_l2_kernel<GA_OP_SUM, int64_t, int32_t, 24, R, U, 4, true, true, true, P1, 0, false, RB>
      <<<(int)p.num_tiles, 24 * 32, 0, s>>>(p, nullptr);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
extern "C" int lab_scan_wide(int v, int64_t n, const void *in, void *out, void *ws, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
    case 0: return run_wide<512, 32, 2, 8>(n, in, out, ws, s);
    case 1: return run_wide<1024, 16, 2, 4>(n, in, out, ws, s);
    case 2: return run_wide<1024, 16, 1, 4>(n, in, out, ws, s);
    case 3: return run_wide<1024, 16, 2, 2>(n, in, out, ws, s);
  }
  return 2;
}

extern "C" int lab_scan(int v, int64_t n, const void *in, void *out, void *ws, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
    case 140: return run_rb<int32_t, 24, 16, 4, 4, 16, 42>(n, in, out, ws, s);
    case 141: return run_rb<int32_t, 24, 16, 4, 8, 16, 42>(n, in, out, ws, s);
    case 142: return run_rb<int32_t, 24, 16, 2, 4, 16, 42>(n, in, out, ws, s);
    case 143: return run_rb<int32_t, 24, 16, 4, 4, 16, 60>(n, in, out, ws, s);
    case 144: return run_rb<int32_t, 24, 16, 4, 4, 16, 30>(n, in, out, ws, s);
    case 145: return run_rb<int32_t, 24, 16, 4, 4, 16, 42, false>(n, in, out, ws, s);
    case 146: return run_rb<int64_t, 24, 16, 2, 4, 16, 42>(n, in, out, ws, s);
    case 147: return run_rb<int64_t, 24, 16, 4, 4, 16, 42>(n, in, out, ws, s);
#define C(id, T, W, R, U, D, P) case id: return run<T, W, R, U, D, P>(n, in, out, ws, s);
    V(C)
#undef C
#define C(id, T, W, R, PF, DIST, U, D, P1) case id: return run<T, W, R, U, D, P1, PF, DIST>(n, in, out, ws, s);
    PFV(C)
#undef C
  }
  return 2;
}
extern "C" int64_t lab_scan_tile(int v) {
  switch (v) {
    case 140:
    case 141:
    case 142:
    case 143:
    case 144:
    case 145: return 24 * 16 * 256;
    case 146:
    case 147: return 24 * 16 * 128;
#define C(id, T, W, R, U, D, P) case id: return (int64_t)W * R * 512 / sizeof(T);
    V(C)
#undef C
#define C(id, T, W, R, PF, DIST, U, D, P1) case id: return (int64_t)W * R * 512 / sizeof(T);
    PFV(C)
#undef C
  }
  return 0;
}
extern "C" int lab_scan_elem_bytes(int v) { return ((v >= 20 && v < 30) || v == 46 || (v >= 50 && v < 140) || v == 146 || v == 147) ? 8 : 4; }

// the product configuration (L shape, int32, exclusive, 32 rows prefetched 42
// ids ahead; v == 1: no prefetch) compiled with TRACE: per tile {start,
// phase 1 done, prefix known, stored, -, -, -, SM id} (tools/lab/trace_l2.py)
extern "C" int lab_scan_trace(int v, int64_t n, const void *in, void *out, void *ws, void *trace, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  constexpr int64_t TILE = 24 * 32 * 512 / 4;
  ScanArgs<int32_t> p = make_args<int32_t>(n, TILE, in, out, nullptr, 0, ws);
  p.pf_dist = v == 1 ? 0 : 42;
  if (v == 1)
    scan_l2_kernel<GA_OP_SUM, int32_t, int32_t, 24, 32, 8, 8, true, true, true, 8, 0, true>
        <<<(int)p.num_tiles, 24 * 32, 0, s>>>(p, (uint64_t *)trace);
  else
    scan_l2_kernel<GA_OP_SUM, int32_t, int32_t, 24, 32, 8, 8, true, true, true, 8, 32, true>
        <<<(int)p.num_tiles, 24 * 32, 0, s>>>(p, (uint64_t *)trace);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// L2 persisting carve-out (device-wide; the evict_last policy lines may live in it)
extern "C" int lab_set_persisting_l2(size_t bytes) {
  cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes);
  size_t got = 0;
  cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
  return e == cudaSuccess ? (int)(got >> 20) : -1;
}
