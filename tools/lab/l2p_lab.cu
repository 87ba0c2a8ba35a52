// l2p_lab.cu — times the product's persistent look-ahead scan kernel shapes.
#include <cuda_runtime.h>
#include <stdint.h>

#include "scan_l2p.cuh"

using namespace ga::scan_detail;

template <typename T, int W, int R, int U, int D, int CPS>
static int run(int64_t n, const void *in, void *out, void *ws, cudaStream_t s) {
  constexpr int64_t TILE = (int64_t)W * R * 512 / sizeof(T);
  ScanArgs<T> p = make_args<T>(n, TILE, in, out, nullptr, 0, ws);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (int64_t)sms * CPS;
  if (grid > p.num_tiles) grid = p.num_tiles;
  scan_l2p_kernel<GA_OP_SUM, T, W, R, U, D, true, true><<<(int)grid, W * 32, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

#define V(X)                               \
  X(0, int32_t, 16, 32, 8, 8, 1)           \
  X(1, int32_t, 24, 32, 8, 8, 1)           \
  X(2, int32_t, 16, 16, 8, 8, 2)           \
  X(3, int32_t, 12, 32, 8, 8, 2)           \
  X(4, int32_t, 16, 24, 8, 8, 1)           \
  X(5, int32_t, 32, 16, 8, 8, 1)           \
  X(6, int32_t, 16, 32, 4, 8, 2)           \
  X(7, int32_t, 8, 32, 8, 8, 3)            \
  X(8, int32_t, 24, 16, 8, 8, 1)           \
  X(20, int64_t, 16, 32, 8, 8, 1)          \
  X(21, int64_t, 24, 32, 8, 8, 1)          \
  X(22, int64_t, 12, 32, 8, 8, 2)

extern "C" int lab_scan(int v, int64_t n, const void *in, void *out, void *ws, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
#define C(id, T, W, R, U, D, CPS) case id: return run<T, W, R, U, D, CPS>(n, in, out, ws, s);
    V(C)
#undef C
  }
  return 2;
}
extern "C" int64_t lab_scan_tile(int v) {
  switch (v) {
#define C(id, T, W, R, U, D, CPS) case id: return (int64_t)W * R * 512 / sizeof(T);
    V(C)
#undef C
  }
  return 0;
}
extern "C" int lab_scan_elem_bytes(int v) { return v >= 20 ? 8 : 4; }
