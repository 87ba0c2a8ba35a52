// scan_lab.cu — tuning lab (not part of the product library): instantiates
// alternative tile shapes of the decoupled look-back scan so one GPU call can
// time them side by side.  Build: see tools/lab/run_scan_lab.py.
#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_variants.cuh"

using namespace ga::scan_lab_old;

static unsigned long long *g_trace = nullptr;
extern "C" void lab_set_trace(void *p) { g_trace = (unsigned long long *)p; }

template <typename T, int BLOCK, int ITEMS, int DEPTH, int BO>
static int run(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  ScanArgs<T> p = make_args<T>(n, (int64_t)BLOCK * ITEMS, in, out, nullptr, 0, ws);
  scan_kernel<T, BLOCK, ITEMS, DEPTH, BO, true, true, true><<<(int)p.num_tiles, BLOCK, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <typename T, int BLOCK, int CH, int STAGES, int DEPTH, int CPS>
static int run_tma(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int TILE_BYTES = BLOCK * CH * 16;
  ScanArgs<T> p = make_args<T>(n, TILE_BYTES / (int)sizeof(T), in, out, nullptr, 0, ws);
  auto k = scan_tma_kernel<T, BLOCK, CH, STAGES, DEPTH, true>;
  const int smem = STAGES * TILE_BYTES;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (int64_t)sms * CPS;
  if (grid > p.num_tiles) grid = p.num_tiles;
  k<<<(int)grid, BLOCK, smem, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <typename T, int BLOCK, int CH, int NSUB, int DEPTH>
static int run_smem(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int TILE_BYTES = BLOCK * CH * 16 * NSUB;
  ScanArgs<T> p = make_args<T>(n, TILE_BYTES / (int)sizeof(T), in, out, nullptr, 0, ws);
  auto k = scan_smem_kernel<T, BLOCK, CH, NSUB, DEPTH, true>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_BYTES);
  k<<<(int)p.num_tiles, BLOCK, TILE_BYTES, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}


template <typename T, int C, int CH, int STAGES, int DEPTH, int NL, int CPS>
static int run_ws(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int TILE_BYTES = C * CH * 512;
  ScanArgs<T> p = make_args<T>(n, TILE_BYTES / (int)sizeof(T), in, out, nullptr, 0, ws);
  p.trace = g_trace;
  auto k = scan_ws_kernel<T, C, CH, STAGES, DEPTH, NL, true>;
  const int smem = STAGES * TILE_BYTES;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (int64_t)sms * CPS;
  if (grid > p.num_tiles) grid = p.num_tiles;
  k<<<(int)grid, (2 + NL + C) * 32, smem, s>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

template <typename T, int WARPS, int ROWS, int UNROLL, int DEPTH, int HINTS>
static int run_l2(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int64_t TILE = (int64_t)WARPS * ROWS * 512 / sizeof(T);
  ScanArgs<T> p = make_args<T>(n, TILE, in, out, nullptr, 0, ws);
  p.trace = g_trace;
  if (HINTS == 2) {  // parked in shared memory
    auto k = scan_l2_kernel<T, WARPS, ROWS, UNROLL, DEPTH, false, true, true, true>;
    const int smem = WARPS * ROWS * 512;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<(int)p.num_tiles, WARPS * 32, smem, s>>>(p);
  } else if (HINTS == 3) {  // parked in shared memory, L2 hints on phase-1 loads
    auto k = scan_l2_kernel<T, WARPS, ROWS, UNROLL, DEPTH, true, true, true, true>;
    const int smem = WARPS * ROWS * 512;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<(int)p.num_tiles, WARPS * 32, smem, s>>>(p);
  } else if (HINTS == 5) {  // early + 2 CTAs/SM forced
    scan_l2_kernel<T, WARPS, ROWS, UNROLL, DEPTH, true, true, true, false, true, 2><<<(int)p.num_tiles, WARPS * 32, 0, s>>>(p);
  } else if (HINTS == 4) {  // early phase-3 loads during the look-back
    scan_l2_kernel<T, WARPS, ROWS, UNROLL, DEPTH, true, true, true, false, true><<<(int)p.num_tiles, WARPS * 32, 0, s>>>(p);
  } else
  scan_l2_kernel<T, WARPS, ROWS, UNROLL, DEPTH, HINTS != 0, true, true><<<(int)p.num_tiles, WARPS * 32, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

template <typename T, int RW, int ROWS, int RU, int WU, int DEPTH>
static int run_pipe(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int64_t TILE = (int64_t)RW * ROWS * 512 / sizeof(T);
  ScanArgs<T> p = make_args<T>(n, TILE, in, out, nullptr, 0, ws);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = sms;
  if (grid > p.num_tiles) grid = p.num_tiles;
  scan_pipe_kernel<T, RW, ROWS, RU, WU, DEPTH, true, true><<<(int)grid, (2 * RW + 1) * 32, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

#define PIPE_VARIANTS(X)                       \
  X(200, int32_t, 8, 64, 16, 8, 4)             \
  X(201, int32_t, 8, 32, 16, 8, 4)             \
  X(202, int32_t, 8, 64, 8, 8, 4)              \
  X(203, int32_t, 12, 32, 16, 8, 4)            \
  X(204, int32_t, 16, 32, 8, 8, 4)             \
  X(205, int32_t, 8, 128, 16, 8, 4)            \
  X(206, int32_t, 16, 16, 16, 8, 4)            \
  X(220, int64_t, 8, 64, 16, 8, 4)             \
  X(221, int64_t, 16, 32, 8, 8, 4)

#define L2_VARIANTS(X)                       \
  X(140, int32_t, 16, 16, 8, 4, 1)           \
  X(141, int32_t, 16, 16, 8, 4, 0)           \
  X(142, int32_t, 16, 32, 8, 4, 1)           \
  X(143, int32_t, 8, 32, 8, 4, 1)            \
  X(144, int32_t, 16, 8, 8, 4, 1)            \
  X(145, int32_t, 32, 16, 8, 4, 1)           \
  X(146, int32_t, 16, 16, 4, 4, 1)           \
  X(147, int32_t, 16, 64, 8, 4, 1)           \
  X(148, int32_t, 16, 32, 8, 4, 0)           \
  X(250, int32_t, 12, 32, 8, 8, 4)           \
  X(251, int32_t, 12, 48, 8, 8, 4)           \
  X(252, int32_t, 12, 64, 8, 8, 4)           \
  X(253, int32_t, 16, 32, 8, 8, 5)           \
  X(254, int32_t, 16, 48, 8, 8, 5)           \
  X(255, int32_t, 8, 64, 8, 8, 4)            \
  X(256, int32_t, 12, 40, 8, 8, 4)           \
  X(257, int64_t, 12, 32, 8, 8, 4)           \
  X(258, int64_t, 12, 48, 8, 8, 4)           \
  X(240, int32_t, 16, 32, 8, 4, 5)           \
  X(241, int32_t, 16, 32, 4, 4, 5)           \
  X(242, int32_t, 32, 16, 4, 4, 4)           \
  X(243, int32_t, 24, 40, 8, 4, 4)           \
  X(244, int32_t, 24, 24, 8, 4, 4)           \
  X(245, int32_t, 32, 16, 8, 4, 4)           \
  X(246, int32_t, 16, 48, 8, 4, 5)           \
  X(247, int32_t, 24, 32, 8, 8, 4)           \
  X(248, int64_t, 24, 32, 8, 4, 4)           \
  X(249, int64_t, 16, 32, 8, 4, 5)           \
  X(230, int32_t, 16, 32, 8, 4, 4)           \
  X(231, int32_t, 16, 24, 8, 4, 4)           \
  X(232, int32_t, 24, 32, 8, 4, 4)           \
  X(233, int32_t, 16, 32, 8, 2, 4)           \
  X(234, int32_t, 16, 16, 8, 4, 4)           \
  X(235, int64_t, 16, 32, 8, 4, 4)           \
  X(236, int64_t, 16, 16, 8, 4, 4)           \
  X(180, int32_t, 16, 32, 8, 8, 1)           \
  X(181, int32_t, 16, 32, 8, 2, 1)           \
  X(182, int32_t, 16, 24, 8, 4, 1)           \
  X(183, int32_t, 16, 40, 8, 4, 1)           \
  X(184, int32_t, 16, 48, 8, 4, 1)           \
  X(185, int32_t, 12, 32, 8, 4, 1)           \
  X(186, int32_t, 20, 32, 8, 4, 1)           \
  X(187, int32_t, 24, 32, 8, 4, 1)           \
  X(188, int32_t, 16, 36, 6, 4, 1)           \
  X(189, int32_t, 16, 30, 10, 4, 1)          \
  X(190, int32_t, 16, 32, 4, 4, 1)           \
  X(149, int32_t, 16, 32, 4, 4, 1)           \
  X(150, int32_t, 16, 64, 4, 4, 1)           \
  X(151, int32_t, 32, 32, 4, 4, 1)           \
  X(152, int32_t, 8, 64, 8, 4, 1)            \
  X(153, int32_t, 16, 32, 16, 4, 1)          \
  X(154, int32_t, 32, 16, 4, 4, 1)           \
  X(155, int32_t, 8, 32, 4, 4, 1)            \
  X(156, int32_t, 16, 32, 8, 1, 1)           \
  X(170, int32_t, 16, 12, 4, 4, 2)           \
  X(171, int32_t, 16, 8, 4, 4, 2)            \
  X(172, int32_t, 8, 24, 8, 4, 2)            \
  X(173, int32_t, 16, 24, 8, 4, 2)           \
  X(174, int32_t, 32, 12, 4, 4, 2)           \
  X(175, int32_t, 8, 16, 8, 4, 2)            \
  X(176, int32_t, 16, 12, 4, 4, 3)           \
  X(177, int32_t, 8, 12, 4, 4, 2)            \
  X(178, int64_t, 16, 12, 4, 4, 2)           \
  X(179, int64_t, 8, 24, 8, 4, 2)            \
  X(160, int64_t, 16, 16, 8, 4, 1)           \
  X(161, int64_t, 16, 32, 8, 4, 1)           \
  X(162, int64_t, 16, 16, 8, 4, 0)

#define WS_VARIANTS(X)                    \
  X(100, int32_t, 8, 8, 6, 4, 2, 1)        \
  X(101, int32_t, 8, 8, 3, 4, 2, 2)        \
  X(102, int32_t, 4, 8, 6, 4, 2, 2)        \
  X(103, int32_t, 8, 16, 3, 4, 2, 1)       \
  X(104, int32_t, 16, 8, 3, 4, 2, 1)       \
  X(105, int32_t, 8, 8, 6, 4, 1, 1)        \
  X(106, int32_t, 8, 8, 6, 8, 3, 1)        \
  X(107, int32_t, 8, 8, 4, 4, 2, 1)        \
  X(120, int64_t, 8, 8, 6, 4, 2, 1)        \
  X(121, int64_t, 8, 8, 3, 4, 2, 2)        \
  X(122, int64_t, 16, 8, 3, 4, 2, 1)

#define SMEM_VARIANTS(X)              \
  X(80, int32_t, 256, 8, 3, 1)         \
  X(81, int32_t, 256, 8, 3, 4)         \
  X(82, int32_t, 256, 8, 2, 1)         \
  X(83, int32_t, 256, 8, 6, 1)         \
  X(84, int32_t, 512, 4, 3, 1)         \
  X(85, int32_t, 256, 4, 3, 1)         \
  X(86, int32_t, 128, 8, 6, 1)         \
  X(87, int32_t, 256, 8, 4, 1)         \
  X(88, int32_t, 256, 8, 2, 8)         \
  X(89, int32_t, 256, 8, 2, 16)        \
  X(79, int32_t, 256, 8, 3, 16)        \
  X(78, int32_t, 256, 8, 6, 16)        \
  X(93, int64_t, 256, 8, 2, 16)        \
  X(90, int64_t, 256, 8, 3, 1)         \
  X(91, int64_t, 256, 8, 2, 1)         \
  X(92, int64_t, 256, 8, 6, 1)

#define TMA_VARIANTS(X)                 \
  X(40, int32_t, 256, 8, 3, 4, 2)        \
  X(41, int32_t, 256, 8, 3, 2, 2)        \
  X(42, int32_t, 256, 8, 6, 4, 1)        \
  X(43, int32_t, 256, 4, 6, 4, 2)        \
  X(44, int32_t, 512, 4, 3, 4, 2)        \
  X(45, int32_t, 256, 8, 2, 4, 3)        \
  X(46, int32_t, 128, 8, 4, 4, 4)        \
  X(47, int32_t, 256, 16, 2, 4, 2)       \
  X(60, int64_t, 256, 8, 3, 4, 2)        \
  X(61, int64_t, 256, 8, 6, 4, 1)        \
  X(62, int64_t, 256, 4, 6, 4, 2)

#define VARIANTS(X)                    \
  X(0, int32_t, 256, 16, 1, 0)         \
  X(1, int32_t, 256, 16, 4, 0)         \
  X(2, int32_t, 256, 16, 4, 100)       \
  X(3, int32_t, 512, 16, 4, 0)         \
  X(4, int32_t, 256, 32, 4, 0)         \
  X(5, int32_t, 512, 32, 4, 0)         \
  X(6, int32_t, 128, 32, 4, 0)         \
  X(7, int32_t, 256, 24, 4, 0)         \
  X(8, int32_t, 1024, 16, 4, 0)        \
  X(9, int32_t, 128, 16, 4, 0)         \
  X(10, int32_t, 512, 8, 4, 0)         \
  X(11, int32_t, 256, 8, 4, 0)         \
  X(20, int64_t, 256, 8, 4, 0)         \
  X(21, int64_t, 256, 16, 4, 0)        \
  X(22, int64_t, 512, 8, 4, 0)         \
  X(23, int64_t, 128, 16, 4, 0)        \
  X(24, int64_t, 256, 8, 1, 0)

extern "C" int lab_scan(int v, int64_t n, const void *in, void *out, void *ws, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
#define CASE(id, T, B, I, D, BO) \
  case id: return run<T, B, I, D, BO>(n, in, out, ws, s);
    VARIANTS(CASE)
#undef CASE
#define PCASE(id, T, RW, R, RU, WU, D) \
  case id: return run_pipe<T, RW, R, RU, WU, D>(n, in, out, ws, s);
    PIPE_VARIANTS(PCASE)
#undef PCASE
#define LCASE(id, T, W, R, U, D, H) \
  case id: return run_l2<T, W, R, U, D, H>(n, in, out, ws, s);
    L2_VARIANTS(LCASE)
#undef LCASE
#define WCASE(id, T, C, CH, S, D, NL, CPS) \
  case id: return run_ws<T, C, CH, S, D, NL, CPS>(n, in, out, ws, s);
    WS_VARIANTS(WCASE)
#undef WCASE
#define SCASE(id, T, B, C, NS, D) \
  case id: return run_smem<T, B, C, NS, D>(n, in, out, ws, s);
    SMEM_VARIANTS(SCASE)
#undef SCASE
#define TCASE(id, T, B, C, S, D, CPS) \
  case id: return run_tma<T, B, C, S, D, CPS>(n, in, out, ws, s);
    TMA_VARIANTS(TCASE)
#undef TCASE
  }
  return 2;
}

extern "C" int64_t lab_scan_tile(int v) {
  switch (v) {
#define TILE(id, T, B, I, D, BO) \
  case id: return (int64_t)B * I;
    VARIANTS(TILE)
#undef TILE
#define PTILE(id, T, RW, R, RU, WU, D) \
  case id: return (int64_t)RW * R * 512 / sizeof(T);
    PIPE_VARIANTS(PTILE)
#undef PTILE
#define LTILE(id, T, W, R, U, D, H) \
  case id: return (int64_t)W * R * 512 / sizeof(T);
    L2_VARIANTS(LTILE)
#undef LTILE
#define WTILE(id, T, C, CH, S, D, NL, CPS) \
  case id: return (int64_t)C * CH * 512 / sizeof(T);
    WS_VARIANTS(WTILE)
#undef WTILE
#define STILE(id, T, B, C, NS, D) \
  case id: return (int64_t)B * C * 16 * NS / sizeof(T);
    SMEM_VARIANTS(STILE)
#undef STILE
#define TTILE(id, T, B, C, S, D, CPS) \
  case id: return (int64_t)B * C * 16 / sizeof(T);
    TMA_VARIANTS(TTILE)
#undef TTILE
  }
  return 0;
}

extern "C" int lab_scan_elem_bytes(int v) { return (v >= 20 && v < 40) || (v >= 60 && v < 78) || (v >= 90 && v < 100) || (v >= 120 && v < 140) || (v >= 160 && v < 170) || (v >= 178 && v < 180) || (v >= 191 && v < 200) || (v >= 220 && v < 230) || v == 235 || v == 236 || v == 248 || v == 249 || v == 257 || v == 258 ? 8 : 4; }
