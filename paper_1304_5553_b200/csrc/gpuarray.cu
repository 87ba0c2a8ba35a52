// gpuarray.cu — the C ABI declared in include/gpuarray.h: argument
// validation, dispatch to the kernel launchers, status strings and
// thread-local error detail.  No device allocation, no host synchronisation.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <utility>

#include "ga_host.h"
#include "gpuarray.h"

namespace ga {

static thread_local char g_last_error[512] = "";
static std::atomic<uint64_t> g_launches{0};

ga_status_t fail(ga_status_t s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return s;
}

ga_status_t check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return GA_OK;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 1;
}

int resident_grid(const void *kernel, int block, size_t dyn_smem) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(kernel, dev * 65536 + block);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, dyn_smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  int grid = per_sm * sm_count();
  cache[key] = grid;
  return grid;
}

// Opt a kernel into `bytes` of dynamic shared memory on the current device,
// once per (kernel, device): function attributes belong to a device's
// context, so a process that drives several GPUs sets them on each.
cudaError_t allow_dyn_smem(const void *kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, cudaError_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(kernel, dev);
  auto it = done.find(key);
  if (it != done.end()) return it->second;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) cudaGetLastError();
  done[key] = e;
  return e;
}

}  // namespace ga

using namespace ga;

static bool scalar_ok(const ga_scalar_t &s, ga_dtype_t dt) { return s.dtype == (int32_t)dt && s.reserved == 0; }

extern "C" {

ga_status_t gpuarray_axpbyz(ga_dtype_t dt, int64_t n, ga_scalar_t a, const void *x, ga_scalar_t b, const void *y,
                            void *z, void *stream) {
  if (!valid_dtype(dt)) return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz: bad dtype %d", (int)dt);
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz: n < 0");
  if (!scalar_ok(a, dt) || !scalar_ok(b, dt))
    return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz: scalar dtype differs from array dtype");
  if (n == 0) return GA_OK;
  if (!x || !y || !z) return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz: NULL array with n > 0");
  const size_t bytes = (size_t)n * dtype_size(dt);
  if (partial_overlap(z, bytes, x, bytes) || partial_overlap(z, bytes, y, bytes))
    return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz: z partially overlaps x or y");
  return launch_axpbyz(dt, n, a, x, b, y, z, (cudaStream_t)stream);
}

ga_status_t gpuarray_axpbyz_ds(ga_dtype_t dt, int64_t n, ga_dscalar_t a, const void *x, ga_dscalar_t b,
                               const void *y, void *z, void *stream) {
  if (!valid_dtype(dt)) return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz_ds: bad dtype %d", (int)dt);
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz_ds: n < 0");
  if (!scalar_ok(a.scale, dt) || !scalar_ok(b.scale, dt))
    return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz_ds: scalar dtype differs from array dtype");
  if (dt != GA_F32 && dt != GA_F64)
    return fail(GA_ERR_UNSUPPORTED, "axpbyz_ds: device-scalar factors need F32 or F64");
  if (n == 0) return GA_OK;
  if (!x || !y || !z) return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz_ds: NULL array with n > 0");
  const size_t bytes = (size_t)n * dtype_size(dt);
  if (partial_overlap(z, bytes, x, bytes) || partial_overlap(z, bytes, y, bytes))
    return fail(GA_ERR_INVALID_ARGUMENT, "axpbyz_ds: z partially overlaps x or y");
  return launch_axpbyz_ds(dt, n, a.scale, a.num, a.den, x, b.scale, b.num, b.den, y, z, (cudaStream_t)stream);
}

ga_status_t gpuarray_axpbz(ga_dtype_t dt, int64_t n, ga_scalar_t a, const void *x, ga_scalar_t b, void *z,
                           void *stream) {
  if (!valid_dtype(dt)) return fail(GA_ERR_INVALID_ARGUMENT, "axpbz: bad dtype %d", (int)dt);
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "axpbz: n < 0");
  if (!scalar_ok(a, dt) || !scalar_ok(b, dt))
    return fail(GA_ERR_INVALID_ARGUMENT, "axpbz: scalar dtype differs from array dtype");
  if (n == 0) return GA_OK;
  if (!x || !z) return fail(GA_ERR_INVALID_ARGUMENT, "axpbz: NULL array with n > 0");
  const size_t bytes = (size_t)n * dtype_size(dt);
  if (partial_overlap(z, bytes, x, bytes)) return fail(GA_ERR_INVALID_ARGUMENT, "axpbz: z partially overlaps x");
  return launch_axpbz(dt, n, a, x, b, z, (cudaStream_t)stream);
}

size_t gpuarray_reduce_workspace_bytes(ga_dtype_t out_dt, int64_t n) {
  (void)out_dt;
  (void)n;
  return reduce_workspace_bytes();
}

ga_status_t gpuarray_reduce(ga_op_t op, ga_map_t map, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n, const void *x,
                            const void *y, void *out, void *workspace, size_t workspace_bytes, void *stream) {
  if (op < GA_OP_SUM || op > GA_OP_MIN) return fail(GA_ERR_INVALID_ARGUMENT, "reduce: bad op %d", (int)op);
  if (map < GA_MAP_ID || map > GA_MAP_CONJ_MUL) return fail(GA_ERR_INVALID_ARGUMENT, "reduce: bad map %d", (int)map);
  if (!valid_dtype(in_dt) || !valid_dtype(out_dt)) return fail(GA_ERR_INVALID_ARGUMENT, "reduce: bad dtype");
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "reduce: n < 0");
  if (!out) return fail(GA_ERR_INVALID_ARGUMENT, "reduce: out is NULL");
  if (n > 0 && !x) return fail(GA_ERR_INVALID_ARGUMENT, "reduce: x is NULL with n > 0");
  const bool has_y = map == GA_MAP_MUL || map == GA_MAP_CONJ_MUL;
  if (has_y && n > 0 && !y) return fail(GA_ERR_INVALID_ARGUMENT, "reduce: MAP_MUL / MAP_CONJ_MUL need y");
  if (!workspace || workspace_bytes < reduce_workspace_bytes())
    return fail(GA_ERR_WORKSPACE, "reduce: workspace needs %zu bytes", reduce_workspace_bytes());
  return launch_reduce(op, map, in_dt, out_dt, n, x, has_y ? y : nullptr, out, workspace, Exchange(),
                       (cudaStream_t)stream);
}

size_t gpuarray_xgpu_buffer_bytes(void) { return (size_t)2 * XG_MAX_WORLD * XG_SLOT; }

ga_status_t gpuarray_reduce_xgpu(ga_op_t op, ga_map_t map, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                                 const void *x, const void *y, void *out, void *workspace, size_t workspace_bytes,
                                 const uint64_t *peer_buffers, int rank, int world, uint64_t seq,
                                 ga_xgpu_fold_t fold, void *stream) {
  if (op < GA_OP_SUM || op > GA_OP_MIN) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: bad op %d", (int)op);
  if (map < GA_MAP_ID || map > GA_MAP_CONJ_MUL) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: bad map");
  if (!valid_dtype(in_dt) || !valid_dtype(out_dt)) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: bad dtype");
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: n < 0");
  if (!out) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: out is NULL");
  if (n > 0 && !x) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: x is NULL with n > 0");
  const bool has_y = map == GA_MAP_MUL || map == GA_MAP_CONJ_MUL;
  if (has_y && n > 0 && !y) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: MAP_MUL / MAP_CONJ_MUL need y");
  if (world < 1 || world > XG_MAX_WORLD || rank < 0 || rank >= world || !peer_buffers || seq == 0)
    return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: bad rank/world/peers/seq");
  if (fold != GA_XGPU_ALL && fold != GA_XGPU_EXCLUSIVE_PREFIX)
    return fail(GA_ERR_INVALID_ARGUMENT, "reduce_xgpu: bad fold %d", (int)fold);
  if (!workspace || workspace_bytes < reduce_workspace_bytes())
    return fail(GA_ERR_WORKSPACE, "reduce_xgpu: workspace needs %zu bytes", reduce_workspace_bytes());
  Exchange xg;
  xg.peers = reinterpret_cast<const unsigned long long *>(peer_buffers);
  xg.rank = rank;
  xg.world = world;
  xg.seq = seq;
  xg.prefix_only = fold == GA_XGPU_EXCLUSIVE_PREFIX;
  return launch_reduce(op, map, in_dt, out_dt, n, x, has_y ? y : nullptr, out, workspace, xg,
                       (cudaStream_t)stream);
}

size_t gpuarray_scan_workspace_bytes(ga_dtype_t dt, int64_t n) { return n < 0 ? 0 : scan_workspace_bytes(dt, n); }

ga_status_t gpuarray_scan(ga_op_t op, ga_scan_kind_t kind, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                          const void *in, void *out, const void *carry, int64_t carry_count, void *workspace,
                          size_t workspace_bytes, void *stream) {
  if (op < GA_OP_SUM || op > GA_OP_MIN) return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad op %d", (int)op);
  if (kind != GA_SCAN_INCLUSIVE && kind != GA_SCAN_EXCLUSIVE)
    return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad kind %d", (int)kind);
  if (!valid_dtype(in_dt) || !valid_dtype(out_dt))
    return fail(GA_ERR_INVALID_ARGUMENT, "scan: bad dtype %d -> %d", (int)in_dt, (int)out_dt);
  if (in_dt == GA_C64 || in_dt == GA_C128 || out_dt == GA_C64 || out_dt == GA_C128)
    return fail(GA_ERR_UNSUPPORTED, "scan: complex not instantiated");
  if (in_dt != out_dt && !((in_dt == GA_I32 && out_dt == GA_I64) || (in_dt == GA_F32 && out_dt == GA_F64)))
    return fail(GA_ERR_UNSUPPORTED, "scan %d -> %d not instantiated (widening: int32 -> int64, float32 -> float64)",
                (int)in_dt, (int)out_dt);
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "scan: n < 0");
  if (carry_count < 0 || (carry_count > 0 && !carry))
    return fail(GA_ERR_INVALID_ARGUMENT, "scan: carry_count < 0 or carry NULL");
  if (n == 0) return GA_OK;
  if (!in || !out) return fail(GA_ERR_INVALID_ARGUMENT, "scan: NULL array with n > 0");
  const size_t in_bytes = (size_t)n * dtype_size(in_dt), out_bytes = (size_t)n * dtype_size(out_dt);
  if (in_dt == out_dt ? partial_overlap(out, out_bytes, in, in_bytes)
                      : (in == out || partial_overlap(out, out_bytes, in, in_bytes)))
    return fail(GA_ERR_INVALID_ARGUMENT, "scan: out overlaps in (a widening scan cannot run in place)");
  const size_t need = scan_workspace_bytes(out_dt, n);
  if (!workspace || workspace_bytes < need) return fail(GA_ERR_WORKSPACE, "scan: workspace needs %zu bytes", need);
  return launch_scan(op, kind, in_dt, out_dt, n, in, out, carry, carry_count, workspace, (cudaStream_t)stream);
}

ga_status_t gpuarray_elementwise(ga_ewop_t op, ga_dtype_t dt, int64_t n, const void *x, const void *y, void *z,
                                 void *stream) {
  if (op < GA_EW_MUL || op > GA_EW_MIN) return fail(GA_ERR_INVALID_ARGUMENT, "elementwise: bad op %d", (int)op);
  if (!valid_dtype(dt)) return fail(GA_ERR_INVALID_ARGUMENT, "elementwise: bad dtype %d", (int)dt);
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "elementwise: n < 0");
  if (n == 0) return GA_OK;
  const bool bin = ewop_binary(op);
  if (!x || !z || (bin && !y)) return fail(GA_ERR_INVALID_ARGUMENT, "elementwise: NULL array with n > 0");
  const size_t bytes = (size_t)n * dtype_size(dt);
  if (partial_overlap(z, bytes, x, bytes) || (bin && partial_overlap(z, bytes, y, bytes)))
    return fail(GA_ERR_INVALID_ARGUMENT, "elementwise: z partially overlaps an input");
  return launch_ewmap(op, dt, n, x, bin ? y : nullptr, z, (cudaStream_t)stream);
}

ga_status_t gpuarray_stencil3(ga_dtype_t dt, int64_t n, ga_scalar_t l, ga_scalar_t d, ga_scalar_t u,
                              const void *diag, const void *x, void *y, void *stream) {
  if (!valid_dtype(dt)) return fail(GA_ERR_INVALID_ARGUMENT, "stencil3: bad dtype %d", (int)dt);
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "stencil3: n < 0");
  if (!scalar_ok(l, dt) || !scalar_ok(d, dt) || !scalar_ok(u, dt))
    return fail(GA_ERR_INVALID_ARGUMENT, "stencil3: scalar dtype differs from array dtype");
  if (n == 0) return GA_OK;
  if (!x || !y) return fail(GA_ERR_INVALID_ARGUMENT, "stencil3: NULL array with n > 0");
  const size_t bytes = (size_t)n * dtype_size(dt);
  if ((uintptr_t)x < (uintptr_t)y + bytes && (uintptr_t)y < (uintptr_t)x + bytes)
    return fail(GA_ERR_INVALID_ARGUMENT, "stencil3: y overlaps x (neighbours are read)");
  if (diag && (uintptr_t)diag < (uintptr_t)y + bytes && (uintptr_t)y < (uintptr_t)diag + bytes)
    return fail(GA_ERR_INVALID_ARGUMENT, "stencil3: y overlaps diag");
  return launch_stencil3(dt, n, l, d, u, diag, x, y, (cudaStream_t)stream);
}

static bool overlaps(const void *p, const void *q, size_t bytes) {
  return p && q && (uintptr_t)p < (uintptr_t)q + bytes && (uintptr_t)q < (uintptr_t)p + bytes;
}

ga_status_t gpuarray_cg_direction(ga_dtype_t dt, int64_t n, ga_dscalar_t beta, const void *r, const void *p_in,
                                  void *p_out, ga_scalar_t l, ga_scalar_t d, ga_scalar_t u, const void *diag, void *ap,
                                  void *pap, void *workspace, size_t workspace_bytes, void *stream) {
  if (!valid_dtype(dt)) return fail(GA_ERR_INVALID_ARGUMENT, "cg_direction: bad dtype %d", (int)dt);
  if (dt != GA_F32 && dt != GA_F64) return fail(GA_ERR_UNSUPPORTED, "cg_direction: F32 or F64 only");
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "cg_direction: n < 0");
  if (!scalar_ok(beta.scale, dt) || !scalar_ok(l, dt) || !scalar_ok(d, dt) || !scalar_ok(u, dt))
    return fail(GA_ERR_INVALID_ARGUMENT, "cg_direction: scalar dtype differs from array dtype");
  if (!pap) return fail(GA_ERR_INVALID_ARGUMENT, "cg_direction: NULL pap");
  if (n > 0 && (!r || !p_in || !p_out || !ap)) return fail(GA_ERR_INVALID_ARGUMENT, "cg_direction: NULL array");
  const size_t bytes = (size_t)n * dtype_size(dt);
  const void *ins[] = {r, p_in, diag};
  for (const void *q : ins)
    if (overlaps(p_out, q, bytes) || overlaps(ap, q, bytes))
      return fail(GA_ERR_INVALID_ARGUMENT, "cg_direction: p_out / ap overlap an input (neighbours are read)");
  if (overlaps(p_out, ap, bytes)) return fail(GA_ERR_INVALID_ARGUMENT, "cg_direction: p_out overlaps ap");
  if (!workspace || workspace_bytes < gpuarray_reduce_workspace_bytes(dt, n))
    return fail(GA_ERR_WORKSPACE, "cg_direction: workspace needs %zu bytes", gpuarray_reduce_workspace_bytes(dt, n));
  return launch_cg_direction(dt, n, beta, r, p_in, p_out, l, d, u, diag, ap, pap, workspace, (cudaStream_t)stream);
}

ga_status_t gpuarray_cg_update(ga_dtype_t dt, int64_t n, ga_dscalar_t alpha, void *x, void *r, const void *p,
                               const void *ap, void *rr, void *workspace, size_t workspace_bytes, void *stream) {
  if (!valid_dtype(dt)) return fail(GA_ERR_INVALID_ARGUMENT, "cg_update: bad dtype %d", (int)dt);
  if (dt != GA_F32 && dt != GA_F64) return fail(GA_ERR_UNSUPPORTED, "cg_update: F32 or F64 only");
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "cg_update: n < 0");
  if (!scalar_ok(alpha.scale, dt)) return fail(GA_ERR_INVALID_ARGUMENT, "cg_update: scalar dtype differs");
  if (!rr) return fail(GA_ERR_INVALID_ARGUMENT, "cg_update: NULL rr");
  if (n > 0 && (!x || !r || !p || !ap)) return fail(GA_ERR_INVALID_ARGUMENT, "cg_update: NULL array");
  const size_t bytes = (size_t)n * dtype_size(dt);
  const void *all[] = {x, r, p, ap};
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j)
      if (overlaps(all[i], all[j], bytes)) return fail(GA_ERR_INVALID_ARGUMENT, "cg_update: x, r, p, ap overlap");
  if (!workspace || workspace_bytes < gpuarray_reduce_workspace_bytes(dt, n))
    return fail(GA_ERR_WORKSPACE, "cg_update: workspace needs %zu bytes", gpuarray_reduce_workspace_bytes(dt, n));
  return launch_cg_update(dt, n, alpha, x, r, p, ap, rr, workspace, (cudaStream_t)stream);
}

const char *gpuarray_status_string(ga_status_t s) {
  switch (s) {
    case GA_OK: return "GA_OK";
    case GA_ERR_INVALID_ARGUMENT: return "GA_ERR_INVALID_ARGUMENT";
    case GA_ERR_UNSUPPORTED: return "GA_ERR_UNSUPPORTED";
    case GA_ERR_WORKSPACE: return "GA_ERR_WORKSPACE";
    case GA_ERR_CUDA: return "GA_ERR_CUDA";
    case GA_ERR_NCCL: return "GA_ERR_NCCL";
  }
  return "GA_ERR_UNKNOWN";
}

const char *gpuarray_last_error(void) { return g_last_error; }

int gpuarray_abi_version(void) { return GPUARRAY_ABI_VERSION; }

uint64_t gpuarray_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
