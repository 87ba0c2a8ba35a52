// smem_lab.cu — tuning lab only (round 2): shapes of the single-touch
// scan_smem_kernel (csrc/scan_smem.cuh): data warps, slice bytes, prefetch.
#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_smem.cuh"

using namespace ga::scan_detail;

template <typename T, int DW, int SLICE, int D, bool EX, bool PF, bool STMA = false, bool SRV = false>
static int run(int64_t n, const void *in, void *out, void *ws, int pfd, cudaStream_t s) {
  constexpr int64_t TILE = (int64_t)DW * SLICE / sizeof(T);
  constexpr int SMEM = DW * SLICE;
  auto k = scan_smem_kernel<GA_OP_SUM, T, DW, SLICE, D, true, EX, PF, false, STMA, SRV>;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    init = true;
  }
  ScanArgs<T> p = make_args<T>(n, TILE, in, out, nullptr, 0, ws);
  p.pf_dist = pfd;
  k<<<(int)p.num_tiles, (DW + 1) * 32, SMEM, s>>>(p, nullptr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

// id, T, data warps, slice bytes, prefetch
#define VS(X)                             \
  X(30, int32_t, 8, 8192, false)          \
  X(31, int32_t, 8, 12288, false)         \
  X(32, int32_t, 8, 8192, true)           \
  X(33, int32_t, 8, 12288, true)          \
  X(34, int32_t, 16, 4096, false)         \
  X(35, int32_t, 8, 4096, false)

#define VSRV(X)                           \
  X(60, int32_t, 8, 12288, false)         \
  X(61, int32_t, 8, 8192, false)          \
  X(62, int32_t, 8, 12288, true)          \
  X(63, int32_t, 8, 8192, true)           \
  X(64, int32_t, 16, 6144, true)          \
  X(65, int32_t, 8, 4096, true)

#define V(X)                              \
  X(0, int32_t, 8, 8192, false)           \
  X(1, int32_t, 16, 4096, false)          \
  X(2, int32_t, 8, 12288, false)          \
  X(3, int32_t, 8, 4096, false)           \
  X(4, int32_t, 16, 6144, false)          \
  X(5, int32_t, 4, 8192, false)           \
  X(6, int32_t, 12, 8192, false)          \
  X(7, int32_t, 8, 6144, false)           \
  X(10, int32_t, 8, 8192, true)           \
  X(11, int32_t, 16, 4096, true)          \
  X(12, int32_t, 8, 12288, true)          \
  X(13, int32_t, 8, 4096, true)           \
  X(20, int64_t, 8, 8192, false)          \
  X(21, int64_t, 16, 4096, false)         \
  X(22, int64_t, 8, 12288, false)         \
  X(23, int64_t, 8, 8192, true)

extern "C" int smem_lab(int v, int ex, int64_t n, const void *in, void *out, void *ws, int pfd, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
#define C(id, T, DW, SL, PF) \
  case id: return ex ? run<T, DW, SL, sizeof(T) == 8 ? 4 : 8, true, PF>(n, in, out, ws, pfd, s) : run<T, DW, SL, sizeof(T) == 8 ? 4 : 8, false, PF>(n, in, out, ws, pfd, s);
    V(C)
#undef C
#define C(id, T, DW, SL, PF) \
  case id: return ex ? run<T, DW, SL, 8, true, PF, true>(n, in, out, ws, pfd, s) : run<T, DW, SL, 8, false, PF, true>(n, in, out, ws, pfd, s);
    VS(C)
#undef C
#define C(id, T, DW, SL, PF) \
  case id: return ex ? run<T, DW, SL, 8, true, PF, false, true>(n, in, out, ws, pfd, s) : run<T, DW, SL, 8, false, PF, false, true>(n, in, out, ws, pfd, s);
    VSRV(C)
#undef C
  }
  return 2;
}
extern "C" int smem_lab_elem_bytes(int v) { return v >= 20 && v < 30 ? 8 : 4; }

// traced runs: per tile {start, loaded, aggregate published, prefix known, stored, -, -, smid}
template <typename T, int DW, int SLICE, bool PF, bool STMA = false>
static int run_trace(int64_t n, const void *in, void *out, void *ws, int pfd, uint64_t *trace, cudaStream_t s) {
  constexpr int64_t TILE = (int64_t)DW * SLICE / sizeof(T);
  constexpr int SMEM = DW * SLICE;
  auto k = scan_smem_kernel<GA_OP_SUM, T, DW, SLICE, 8, true, true, PF, true, STMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  ScanArgs<T> p = make_args<T>(n, TILE, in, out, nullptr, 0, ws);
  p.pf_dist = pfd;
  k<<<(int)p.num_tiles, (DW + 1) * 32, SMEM, s>>>(p, trace);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
extern "C" int smem_lab_trace(int v, int64_t n, const void *in, void *out, void *ws, int pfd, void *trace, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t *tr = (uint64_t *)trace;
  switch (v) {
    case 0: return run_trace<int32_t, 8, 8192, false>(n, in, out, ws, pfd, tr, s);
    case 12: return run_trace<int32_t, 8, 12288, true>(n, in, out, ws, pfd, tr, s);
    case 2: return run_trace<int32_t, 8, 12288, false>(n, in, out, ws, pfd, tr, s);
    case 30: return run_trace<int32_t, 8, 8192, false, true>(n, in, out, ws, pfd, tr, s);
    case 33: return run_trace<int32_t, 8, 12288, true, true>(n, in, out, ws, pfd, tr, s);
  }
  return 2;
}
