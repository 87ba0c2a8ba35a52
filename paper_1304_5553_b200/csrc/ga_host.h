// ga_host.h — host-side helpers of the C ABI: status/error reporting, device
// queries cached per device, launch accounting.  Product code only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpuarray.h"

namespace ga {

// Record a detail string for gpuarray_last_error() and return `s`.
ga_status_t fail(ga_status_t s, const char *fmt, ...);
// Map a CUDA error from a launch to GA_ERR_CUDA (clearing the sticky-free error).
ga_status_t check_launch(const char *what);
// Number of SMs of the current device (cached).
int sm_count();
// Count one kernel launch (gpuarray_launch_count()).
void count_launch();

// Largest grid whose CTAs are all co-resident: SMs x occupancy (cached per
// kernel by the caller through a function-local static).
int resident_grid(const void *kernel, int block, size_t dyn_smem = 0);

// Opt `kernel` into `bytes` of dynamic shared memory on the current device
// (cached per kernel and device).
cudaError_t allow_dyn_smem(const void *kernel, size_t bytes);

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Launch `kernel` on stream s with programmatic stream serialization (PDL):
// the kernel may begin launching before the previous grid in the stream has
// finished; its pdl_enter() (ga_device.cuh) waits for that grid before any
// memory access.  The error, if any, is left for check_launch().
template <typename... Params, typename... Args>
inline void launch(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<Params>(args)...);
}

inline size_t dtype_size(ga_dtype_t dt) {
  return (dt == GA_F32 || dt == GA_I32) ? 4 : dt == GA_C128 ? 16 : 8;
}

inline bool valid_dtype(int dt) { return dt >= GA_F32 && dt <= GA_C128; }

// [p, p+bytes) and [q, q+bytes2) overlap without being the same start.
inline bool partial_overlap(const void *p, size_t bytes, const void *q, size_t bytes2) {
  uintptr_t a = (uintptr_t)p, b = (uintptr_t)q;
  if (a == b) return false;
  return a < b + bytes2 && b < a + bytes;
}

// Cross-GPU finish of a reduction (gpuarray_reduce_xgpu): device array of
// `world` exchange-buffer pointers (one per rank, NVLink-mapped), own rank,
// and the call's sequence number (identical on all ranks, >= 1).
constexpr int XG_MAX_WORLD = 64;
constexpr int XG_SLOT = 32;  // bytes per exchange slot: value (<= 16 B) + seq at +16
struct Exchange {
  const unsigned long long *peers = nullptr;
  int rank = 0;
  int world = 0;
  unsigned long long seq = 0;
  int prefix_only = 0;  // 1: fold only ranks < rank (a sharded scan's offset)
};

// Launchers implemented per kernel family (elementwise.cu, reduce.cu, scan.cu).
ga_status_t launch_axpbyz(ga_dtype_t dt, int64_t n, const ga_scalar_t &a, const void *x,
                          const ga_scalar_t &b, const void *y, void *z, cudaStream_t s);
ga_status_t launch_axpbyz_ds(ga_dtype_t dt, int64_t n, const ga_scalar_t &a, const void *an, const void *ad,
                             const void *x, const ga_scalar_t &b, const void *bn, const void *bd, const void *y,
                             void *z, cudaStream_t s);
ga_status_t launch_axpbz(ga_dtype_t dt, int64_t n, const ga_scalar_t &a, const void *x,
                         const ga_scalar_t &b, void *z, cudaStream_t s);
ga_status_t launch_reduce(ga_op_t op, ga_map_t map, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                          const void *x, const void *y, void *out, void *ws, const Exchange &xg, cudaStream_t s);
ga_status_t launch_scan(ga_op_t op, ga_scan_kind_t kind, ga_dtype_t in_dt, ga_dtype_t dt, int64_t n, const void *in,
                        void *out,
                        const void *carry, int64_t carry_count, void *ws, cudaStream_t s);

ga_status_t launch_stencil3(ga_dtype_t dt, int64_t n, const ga_scalar_t &l, const ga_scalar_t &d,
                            const ga_scalar_t &u, const void *diag, const void *x, void *y, cudaStream_t s);

ga_status_t launch_cg_direction(ga_dtype_t dt, int64_t n, const ga_dscalar_t &beta, const void *r, const void *pin,
                                void *pout, const ga_scalar_t &l, const ga_scalar_t &d, const ga_scalar_t &u,
                                const void *diag, void *ap, void *pap, void *ws, cudaStream_t s);
ga_status_t launch_cg_update(ga_dtype_t dt, int64_t n, const ga_dscalar_t &alpha, void *x, void *r, const void *p,
                             const void *ap, void *rr, void *ws, cudaStream_t s);
bool ewop_binary(ga_ewop_t op);
ga_status_t launch_ewmap(ga_ewop_t op, ga_dtype_t dt, int64_t n, const void *x, const void *y, void *z,
                         cudaStream_t s);

size_t reduce_workspace_bytes();
size_t scan_workspace_bytes(ga_dtype_t dt, int64_t n);

}  // namespace ga
