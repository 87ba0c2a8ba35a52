// sharded.cu — the sharded entry points of the C ABI (SURVEY.md §8(a) a6/a7,
// §8(b)): one call per rank over its contiguous shard, the cross-GPU step an
// NCCL collective on the caller's stream with the caller's communicator.
//
//   gpuarray_reduce_sharded  local single-pass reduce (reduce.cu) of the
//       shard into *out, then ncclAllReduce(out, out, count 1, op) in place:
//       every rank ends with the same bits (BASELINE.json north_star:
//       "Reductions combine per-GPU partials with one NCCL allreduce").
//   gpuarray_scan_sharded    local reduce of the shard -> its total T_g;
//       ncclAllGather of the G totals; local single-pass scan whose carry-in
//       is c ⊕ T_0 ⊕ ... ⊕ T_{g-1} (c the caller's carry), folded into tile 0
//       of the scan kernel ("an exclusive scan of per-GPU totals followed by
//       a local offset add", north_star; R18: 3 element-sizes of
//       HBM traffic per element instead of the 4 of scan-then-add).
//
// NCCL is not linked: the library binds ncclAllReduce / ncclAllGather /
// ncclCommCount / ncclCommUserRank / ncclGetErrorString at the first sharded
// call from the libnccl.so.2 already loaded in the process (the one that
// created the caller's communicator, e.g. torch's ProcessGroupNCCL), else
// loads libnccl.so.2 itself ($GPUARRAY_NCCL_LIB overrides the name).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <mutex>

#include "ga_host.h"
#include "gpuarray.h"

namespace ga {
namespace {

struct NcclApi {
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*count)(const ncclComm_t, int *);
  ncclResult_t (*user_rank)(const ncclComm_t, int *);
  const char *(*error_string)(ncclResult_t);
  bool ok;
  char why[256];
};

const NcclApi &nccl() {
  static NcclApi api{};
  static std::once_flag once;
  std::call_once(once, [] {
    const char *name = getenv("GPUARRAY_NCCL_LIB");
    if (!name || !*name) name = "libnccl.so.2";
    void *h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);  // the instance that made the caller's comm
    if (!h) h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(api.why, sizeof(api.why), "cannot load %s: %s", name, dlerror());
      return;
    }
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.count = reinterpret_cast<decltype(api.count)>(dlsym(h, "ncclCommCount"));
    api.user_rank = reinterpret_cast<decltype(api.user_rank)>(dlsym(h, "ncclCommUserRank"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.all_reduce && api.all_gather && api.count && api.user_rank && api.error_string;
    if (!api.ok) snprintf(api.why, sizeof(api.why), "%s lacks an NCCL entry point", name);
  });
  return api;
}

ga_status_t nccl_fail(const NcclApi &api, const char *what, ncclResult_t r) {
  return fail(GA_ERR_NCCL, "%s: %s", what, api.error_string ? api.error_string(r) : "NCCL error");
}

// NCCL element type and count of one value of dt (complex: 2 reals, SUM only).
bool nccl_type(ga_dtype_t dt, ncclDataType_t &t, size_t &count) {
  count = 1;
  switch (dt) {
    case GA_F32: t = ncclFloat32; return true;
    case GA_F64: t = ncclFloat64; return true;
    case GA_I32: t = ncclInt32; return true;
    case GA_I64: t = ncclInt64; return true;
    case GA_C64: t = ncclFloat32; count = 2; return true;
    case GA_C128: t = ncclFloat64; count = 2; return true;
  }
  return false;
}

ncclRedOp_t nccl_op(ga_op_t op) { return op == GA_OP_MAX ? ncclMax : op == GA_OP_MIN ? ncclMin : ncclSum; }

// Sharded-scan workspace: [reduce workspace | carries: c, T_0 .. T_{G-1} and
// the own total, SHARD_MAX_WORLD + 2 slots of 8 bytes | scan workspace at the
// next 256-byte boundary].  The reduce and scan regions keep their own epochs.
constexpr int SHARD_MAX_WORLD = 4096;
constexpr size_t CARRY_SLOT = 8;  // the scans' largest element
size_t carries_off() { return reduce_workspace_bytes(); }
size_t scan_ws_off() { return (carries_off() + (size_t)(SHARD_MAX_WORLD + 2) * CARRY_SLOT + 255) / 256 * 256; }

}  // namespace
}  // namespace ga

using namespace ga;

extern "C" {

ga_status_t gpuarray_reduce_sharded(ga_op_t op, ga_map_t map, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                                    const void *x, const void *y, void *out, void *workspace, size_t workspace_bytes,
                                    void *nccl_comm, void *stream) {
  if (!nccl_comm) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_sharded: nccl_comm is NULL");
  if ((in_dt == GA_C64 || in_dt == GA_C128) && op != GA_OP_SUM)
    return fail(GA_ERR_UNSUPPORTED, "reduce_sharded: complex needs SUM");
  const NcclApi &api = nccl();
  if (!api.ok) return fail(GA_ERR_NCCL, "reduce_sharded: %s", api.why);
  ga_status_t st = gpuarray_reduce(op, map, in_dt, out_dt, n, x, y, out, workspace, workspace_bytes, stream);
  if (st != GA_OK) return st;
  ncclDataType_t t;
  size_t count;
  if (!nccl_type(out_dt, t, count)) return fail(GA_ERR_INVALID_ARGUMENT, "reduce_sharded: bad out dtype");
  ncclResult_t r = api.all_reduce(out, out, count, t, nccl_op(op), static_cast<ncclComm_t>(nccl_comm),
                                  static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_fail(api, "reduce_sharded: ncclAllReduce", r);
  return GA_OK;
}

size_t gpuarray_scan_sharded_workspace_bytes(ga_dtype_t out_dt, int64_t n) {
  return n < 0 ? 0 : scan_ws_off() + scan_workspace_bytes(out_dt, n);
}

ga_status_t gpuarray_scan_sharded(ga_op_t op, ga_scan_kind_t kind, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                                  const void *in, void *out, const void *carry, int64_t carry_count, void *workspace,
                                  size_t workspace_bytes, void *nccl_comm, void *stream) {
  if (!nccl_comm) return fail(GA_ERR_INVALID_ARGUMENT, "scan_sharded: nccl_comm is NULL");
  if (n < 0) return fail(GA_ERR_INVALID_ARGUMENT, "scan_sharded: n < 0");
  if (carry_count < 0 || (carry_count > 0 && !carry))
    return fail(GA_ERR_INVALID_ARGUMENT, "scan_sharded: carry_count < 0 or carry NULL");
  if (in_dt != out_dt && op != GA_OP_SUM)
    return fail(GA_ERR_UNSUPPORTED, "scan_sharded: widening MAX/MIN scans are not instantiated");
  const size_t need = gpuarray_scan_sharded_workspace_bytes(out_dt, n);
  if (!workspace || workspace_bytes < need)
    return fail(GA_ERR_WORKSPACE, "scan_sharded: workspace needs %zu bytes", need);
  const NcclApi &api = nccl();
  if (!api.ok) return fail(GA_ERR_NCCL, "scan_sharded: %s", api.why);
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int world = 0, rank = 0;
  ncclResult_t r = api.count(comm, &world);
  if (r == ncclSuccess) r = api.user_rank(comm, &rank);
  if (r != ncclSuccess) return nccl_fail(api, "scan_sharded: communicator query", r);
  if (world < 1 || world > SHARD_MAX_WORLD || rank < 0 || rank >= world)
    return fail(GA_ERR_UNSUPPORTED, "scan_sharded: world size %d not supported", world);
  ncclDataType_t t;
  size_t count;
  if (!nccl_type(out_dt, t, count) || count != 1)
    return fail(GA_ERR_UNSUPPORTED, "scan_sharded: dtype %d not instantiated", (int)out_dt);

  char *ws = static_cast<char *>(workspace);
  char *carries = ws + carries_off();           // [c, T_0, ..., T_{G-1}, own total]
  const size_t osz = dtype_size(out_dt);
  char *totals = carries + osz;                 // T_0 .. T_{G-1}
  char *own = totals + (size_t)world * osz;     // this shard's total
  void *scan_ws = ws + scan_ws_off();
  const size_t scan_ws_bytes = workspace_bytes - scan_ws_off();
  // 1. this shard's total, in out_dt (the scan's type: int32 -> int64 and
  //    float32 -> float64 widen on load, like the scan)
  ga_status_t st = gpuarray_reduce(op, GA_MAP_ID, in_dt, out_dt, n, in, nullptr, own, ws, reduce_workspace_bytes(),
                                   stream);
  if (st != GA_OK) return st;
  // 2. every rank's total
  r = api.all_gather(own, totals, 1, t, comm, static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_fail(api, "scan_sharded: ncclAllGather", r);
  // 3. carry-in = c ⊕ T_0 ⊕ ... ⊕ T_{rank-1}: the caller's carries are folded
  //    into one value first (a reduce of the carry array) when there are any
  const void *cptr = totals;
  int64_t ccount = rank;
  if (carry_count > 0) {
    st = gpuarray_reduce(op, GA_MAP_ID, out_dt, out_dt, carry_count, carry, nullptr, carries, ws,
                         reduce_workspace_bytes(), stream);
    if (st != GA_OK) return st;
    cptr = carries;
    ccount = rank + 1;
  }
  // 4. the local scan with that carry-in
  return gpuarray_scan(op, kind, in_dt, out_dt, n, in, out, ccount ? cptr : nullptr, ccount, scan_ws, scan_ws_bytes,
                       stream);
}

}  // extern "C"
