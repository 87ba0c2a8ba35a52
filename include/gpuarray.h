/* gpuarray.h — C ABI of the B200-native GPUArray hot path (arXiv 1304.5553).
 *
 * The three operations of the paper's GPUArray layer, each as one
 * asynchronous call that enqueues ONE hand-written sm_100a kernel on a
 * caller-supplied CUDA stream and returns at once ("the invocation returns
 * immediately and does not wait for completion on the GPU", PAPER.md:338-340,
 * §3.1):
 *
 *   gpuarray_axpbyz / gpuarray_axpbz   ElementwiseKernel, §3.2.4
 *       "a statement ... to be executed for each value of
 *       i ... All these instances are required to have the same length."
 *       The statement is fixed at build time to z[i] = a*x[i] + b*y[i]
 *       (resp. a*x[i] + b) instead of a run-time C string.
 *   gpuarray_reduce                    ReductionKernel (map-reduce), §3.2.5
 *       result dtype (471-472), a map expression over i
 *       (473-477), a reduction expression of a and b with its neutral element
 *       (479-485), result "a GPUArray scalar still residing on the GPU"
 *       (489-492).  The map and reduction expressions are enums.
 *   gpuarray_scan                      parallel prefix sum, §3.2.6
 *       "GPU-based parallel prefix sums".
 *
 * Sharded over GPUs (BASELINE.json north_star):
 *   gpuarray_reduce_sharded / gpuarray_scan_sharded  one call per rank on
 *       its contiguous shard; the cross-GPU step is an NCCL collective on the
 *       caller's stream and communicator.
 *
 * Beyond them: the other GPUArray operators and cumath maps
 * (gpuarray_elementwise), device-scalar coefficients (gpuarray_axpbyz_ds),
 * the fused cross-GPU finish (gpuarray_reduce_xgpu), and the CG workload's
 * operator and fused iteration steps (gpuarray_stencil3, gpuarray_cg_direction,
 * gpuarray_cg_update; the paper's Krylov solver).
 *
 * Conventions (all entry points):
 *   - Pointers x, y, z, in, out, carry, workspace are DEVICE pointers on the
 *     current CUDA device; `stream` is a cudaStream_t (NULL = legacy default
 *     stream).  Arrays are contiguous, 1-D, of n elements of the given dtype,
 *     element-aligned (any offset; the fast path wants x, y, z to share their
 *     address phase modulo 32 bytes — otherwise a slower GPU path is used).
 *   - Ownership: the caller owns every buffer and must keep it alive until
 *     the stream has passed the call.  The library allocates no device
 *     memory, keeps no pointer after returning, and never synchronises.
 *   - Errors (PAPER.md:288-290 raise-on-error model, as status codes): the
 *     return value reports argument and launch errors synchronously; faults
 *     during execution surface at the caller's next synchronisation.
 *     gpuarray_last_error() gives a thread-local detail string.
 *   - Exactly one kernel is launched per call (zero for n == 0, except reduce,
 *     which writes the neutral element with one tiny kernel).
 */
#ifndef GPUARRAY_H
#define GPUARRAY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPUARRAY_ABI_VERSION 5

/* C64 / C128: complex numbers as interleaved (re, im) float / double pairs
 * ("seamless support for complex numbers"; §8(f) NEXT-3). */
typedef enum { GA_F32 = 0, GA_F64 = 1, GA_I32 = 2, GA_I64 = 3, GA_C64 = 4, GA_C128 = 5 } ga_dtype_t;

/* Reduction expression "a+b", "max(a,b)", "min(a,b)" with its neutral element
 * (PAPER.md:479-485 and footnote): SUM 0; MAX -inf / INT_MIN; MIN +inf /
 * INT_MAX (R5).  Floats use maxNum/minNum: a NaN operand loses (R6). */
typedef enum { GA_OP_SUM = 0, GA_OP_MAX = 1, GA_OP_MIN = 2 } ga_op_t;

/* Map expression over index i:
 * x[i] | x[i]*y[i] (dot) | x[i]*x[i] (squared 2-norm; |x[i]|^2 for complex) |
 * conj(x[i])*y[i] (vdot, complex only). */
typedef enum { GA_MAP_ID = 0, GA_MAP_MUL = 1, GA_MAP_SQUARE = 2, GA_MAP_CONJ_MUL = 3 } ga_map_t;

typedef enum { GA_SCAN_INCLUSIVE = 0, GA_SCAN_EXCLUSIVE = 1 } ga_scan_kind_t;

typedef enum {
  GA_OK = 0,
  GA_ERR_INVALID_ARGUMENT = 1, /* n < 0, NULL with n > 0, bad enum, scalar dtype != dt,
                                  y missing for MAP_MUL, partial overlap of output and input */
  GA_ERR_UNSUPPORTED = 2,      /* combination not instantiated (e.g. MAX with out_dt != in_dt) */
  GA_ERR_WORKSPACE = 3,        /* workspace NULL or smaller than *_workspace_bytes() */
  GA_ERR_CUDA = 4,             /* CUDA error at launch; see gpuarray_last_error() */
  GA_ERR_NCCL = 5              /* NCCL missing or a collective failed to enqueue (sharded calls) */
} ga_status_t;

/* A host scalar typed like the arrays it combines with ("numpy sized
 * scalars such as numpy.float32(5.7)"; R2). */
typedef struct ga_scalar {
  int32_t dtype;    /* ga_dtype_t of the value; must equal the call's dt */
  int32_t reserved; /* must be 0 */
  union {
    float f32;
    double f64;
    int32_t i32;
    int64_t i64;
    float c64[2];   /* re, im */
    double c128[2]; /* re, im */
  } v;
} ga_scalar_t;

/* z[i] = a*x[i] + b*y[i], i in [0, n).
 * Floats: z_i = RN(RN(a*x_i) + RN(b*y_i)) — two roundings of the products and
 * one of the sum, no FMA contraction (R1).  Integers wrap modulo
 * 2^w (R4).  Complex: the products written out component-wise with every
 * operation rounded (R24).  dt: any ga_dtype_t.  z may equal x or y exactly
 * (in-place); any other overlap is GA_ERR_INVALID_ARGUMENT.  n == 0: no-op. */
ga_status_t gpuarray_axpbyz(ga_dtype_t dt, int64_t n, ga_scalar_t a, const void *x, ga_scalar_t b,
                            const void *y, void *z, void *stream);

/* A coefficient that may live on the GPU (a reduction's
 * GPUArray scalar "used in-place on the GPU"): value = scale when num and
 * den are both NULL, else RN(scale * RN(num / den)) with a NULL pointer
 * standing for 1 and a zero numerator giving 0 whatever den (0/0 -> 0).  num / den are DEVICE scalars of the call's dt, read when
 * the kernel runs — so a chain of calls (e.g. a CG iteration) needs no host
 * round trip and can be captured in a CUDA graph. */
typedef struct ga_dscalar {
  ga_scalar_t scale;
  const void *num;
  const void *den;
} ga_dscalar_t;

/* axpbyz with device-resident coefficient factors; dt in {F32, F64}; same
 * rounding sequence, overlap rules and n == 0 behaviour as gpuarray_axpbyz. */
ga_status_t gpuarray_axpbyz_ds(ga_dtype_t dt, int64_t n, ga_dscalar_t a, const void *x, ga_dscalar_t b,
                               const void *y, void *z, void *stream);

/* z[i] = a*x[i] + b (floats: RN(RN(a*x_i) + b)).  Listing 1's "multiply by
 * two" is a = 2, b = -0.0 (the IEEE additive identity, R21). */
ga_status_t gpuarray_axpbz(ga_dtype_t dt, int64_t n, ga_scalar_t a, const void *x, ga_scalar_t b,
                           void *z, void *stream);

/* ---- The other GPUArray operators and cumath-style maps (SURVEY.md §8(f)
 * NEXT-2; "support all arithmetic operators ... many special functions are
 * available in pycuda.cumath").  Binary: z = x*y, x/y,
 * maxNum(x,y), minNum(x,y); unary (y ignored, may be NULL): sqrt, |x|, -x,
 * exp, log, sin, cos.  F32/F64: MUL, DIV, SQRT, ABS, NEG, MAX, MIN are IEEE
 * round-to-nearest (bit-exact against the oracle); EXP, LOG, SIN, COS are
 * CUDA's accurate device functions (R26: within a few ulp of
 * glibc).  I32/I64: MUL (wrapping), ABS, NEG (wrapping at INT_MIN), MAX, MIN;
 * others GA_ERR_UNSUPPORTED.  z may equal x or y; n == 0: no-op. */
typedef enum {
  GA_EW_MUL = 0, GA_EW_DIV = 1, GA_EW_SQRT = 2, GA_EW_ABS = 3, GA_EW_NEG = 4, GA_EW_EXP = 5,
  GA_EW_LOG = 6, GA_EW_SIN = 7, GA_EW_COS = 8, GA_EW_MAX = 9, GA_EW_MIN = 10
} ga_ewop_t;
ga_status_t gpuarray_elementwise(ga_ewop_t op, ga_dtype_t dt, int64_t n, const void *x, const void *y, void *z,
                                 void *stream);

/* Bytes of workspace gpuarray_reduce needs (an upper bound for every n and
 * every device).  The workspace must be zero-filled ONCE when allocated; the
 * kernel leaves it reusable (block partials sit in slots tagged with a call
 * epoch that the finishing block advances; a slot is ready when it carries
 * the current call's tag — no reset, no atomics) until the 31-bit tag
 * wraps: zero it again within 2^31 calls (the Python binding counts calls
 * and does).  Calls that may run concurrently need distinct workspaces, and
 * a reduce workspace must not be passed to gpuarray_scan (or vice versa):
 * the layouts differ. */
size_t gpuarray_reduce_workspace_bytes(ga_dtype_t out_dt, int64_t n);

/* *out = fold over i in [0, n) of map(x, y)[i] with `op`, starting from the
 * neutral element; out is a DEVICE scalar of out_dt.
 * Supported (in_dt -> out_dt):
 *   SUM: F32->F32, F32->F64, F64->F64, I32->I32, I32->I64, I64->I64
 *        (accumulation in out_dt; integer maps widen to out_dt then wrap, R3/R4)
 *   SUM over complex: C64->C64, C128->C128 with MAP_ID / MAP_MUL (dot) /
 *        MAP_CONJ_MUL (vdot); MAP_SQUARE gives sum |x|^2: C64->F32, C128->F64
 *   MAX, MIN: real dtypes, out_dt == in_dt; the map is evaluated in in_dt
 *        (RN(x*y), wrap).
 * y must be non-NULL iff map is MAP_MUL or MAP_CONJ_MUL (ignored otherwise).
 * Float SUM is a tree-ordered sum (not the exact sum): deterministic for a
 * given (n, device), accurate as DESIGN.md R9/R10 state.  n == 0 writes the
 * neutral element. */
ga_status_t gpuarray_reduce(ga_op_t op, ga_map_t map, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                            const void *x, const void *y, void *out, void *workspace,
                            size_t workspace_bytes, void *stream);

/* ---- Fused cross-GPU finish (§8(a) a6 in one kernel).
 * Bytes of the per-rank exchange buffer gpuarray_reduce_xgpu needs (2 x 64
 * slots of 32 bytes).  Every rank allocates one in memory all ranks can
 * address (torch symmetric memory over NVLink / NVSwitch), zero-filled once. */
size_t gpuarray_xgpu_buffer_bytes(void);   /* 2 x 64 slots of 32 bytes */

/* What the cross-GPU finish folds: every rank's result (a global reduction),
 * or only the ranks before this one, in rank order (the exclusive prefix over
 * ranks: a sharded scan's carry-in, §8(a) a7).  Rank 0's exclusive prefix is
 * the neutral element. */
typedef enum { GA_XGPU_ALL = 0, GA_XGPU_EXCLUSIVE_PREFIX = 1 } ga_xgpu_fold_t;

/* gpuarray_reduce over a sharded array in ONE kernel per rank: the block that
 * finishes the local reduction stores the local result into slot `rank` of
 * every rank's exchange buffer (peer stores over NVLink, st.release.sys on a
 * sequence word), waits until all `world` slots of its own buffer carry
 * `seq`, and folds them (all, or only ranks < rank: see ga_xgpu_fold_t) in
 * rank order into *out — so every rank ends with the same bits and no
 * separate collective is launched.
 *   peer_buffers  DEVICE array of `world` device pointers; [r] = rank r's
 *                 exchange buffer as mapped on this device
 *   rank, world   1 <= world <= 64
 *   seq           call sequence number, >= 1, identical on all ranks for the
 *                 same logical call and increasing by one per call
 * Everything else as gpuarray_reduce.  All ranks must make the call (a rank
 * that never arrives makes the others trap after 10 s instead of hanging). */
ga_status_t gpuarray_reduce_xgpu(ga_op_t op, ga_map_t map, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                                 const void *x, const void *y, void *out, void *workspace, size_t workspace_bytes,
                                 const uint64_t *peer_buffers, int rank, int world, uint64_t seq,
                                 ga_xgpu_fold_t fold, void *stream);

/* Bytes of workspace gpuarray_scan needs for (dt, n), dt = the scan's OUTPUT
 * dtype: a 256-byte header plus per-tile look-back status.  Zero-fill once;
 * reusable afterwards by scans of any dtype, size and kernel (status words
 * are epoch-tagged, the tile counter resets itself) until the 30-bit call
 * epoch wraps: zero it again within 2^30 calls (the Python binding counts
 * calls and does).  One call at a time per workspace: calls that may run
 * concurrently (different streams) need their own.  Never share it with
 * gpuarray_reduce.  A corrupted workspace makes the kernel trap (a CUDA
 * error at the next synchronisation) after 10 s instead of hanging. */
size_t gpuarray_scan_workspace_bytes(ga_dtype_t dt, int64_t n);

/* Scan (§3.2.6 "parallel prefix sums") with the reduction
 * expression op ∈ {SUM, MAX, MIN} (written ⊕ below):
 *   inclusive: out[i] = c ⊕ w(in[0]) ⊕ ... ⊕ w(in[i])
 *   exclusive: out[0] = c, out[i] = c ⊕ w(in[0]) ⊕ ... ⊕ w(in[i-1])   (R13)
 * in_dt == out_dt ∈ {F32, F64, I32, I64}, or the widening scans in_dt = I32,
 * out_dt = I64 and in_dt = F32, out_dt = F64 (NEXT-2; the paper makes the
 * result dtype a parameter); w() is the exact conversion to out_dt
 * and the scan runs in out_dt.  Other pairs and complex: GA_ERR_UNSUPPORTED.
 * c = carry[0] ⊕ ... ⊕ carry[carry_count-1] is a device array of out_dt (the
 * neutral element when carry_count == 0); it is how a sharded scan passes
 * the totals of earlier shards.  Integers wrap (R4,
 * R14); MAX/MIN are exact (maxNum/minNum for floats, R6); float SUM is a
 * tree/look-back-ordered approximation of the exact prefix sums (DESIGN.md
 * R22), not bit-reproducible run to run.  in: n elements of in_dt; out: n
 * elements of out_dt.  out may equal in when in_dt == out_dt (in-place);
 * any other overlap is GA_ERR_INVALID_ARGUMENT.  n == 0: no-op. */
ga_status_t gpuarray_scan(ga_op_t op, ga_scan_kind_t kind, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                          const void *in, void *out, const void *carry, int64_t carry_count, void *workspace,
                          size_t workspace_bytes, void *stream);

/* ---- Sharded over GPUs (BASELINE.json
 * north_star: "Arrays are sharded contiguously ... Reductions combine per-GPU
 * partials with one NCCL allreduce over NVLink.  Scan uses an exclusive scan
 * of per-GPU totals followed by a local offset add").  One call per rank, on
 * the rank's contiguous shard [start_g, start_g + n) of the global array
 * (start_g = floor(g*N/G), R16), with every rank making the same
 * sequence of sharded calls (collective semantics).
 *   nccl_comm  an initialised ncclComm_t (e.g. torch's
 *              ProcessGroupNCCL._comm_ptr()), whose rank order is the shard
 *              order; NCCL is bound at run time from the libnccl.so.2 already
 *              loaded in the process (else loaded; $GPUARRAY_NCCL_LIB).  A
 *              missing NCCL or a failed enqueue returns GA_ERR_NCCL.
 * The collective runs on `stream` after the local kernel; nothing is
 * synchronised.  Results are identical on every rank. */

/* gpuarray_reduce over the global array: the local single-pass reduction of
 * the shard into *out (every argument as gpuarray_reduce; `workspace` is a
 * gpuarray_reduce workspace), then ONE ncclAllReduce(out, out, 1 value, op)
 * in place (SUM / MAX / MIN; complex: SUM of the 2 components).  Float SUM:
 * the local tree sum, then NCCL's fixed-topology combine (R17). */
ga_status_t gpuarray_reduce_sharded(ga_op_t op, ga_map_t map, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                                    const void *x, const void *y, void *out, void *workspace, size_t workspace_bytes,
                                    void *nccl_comm, void *stream);

/* Bytes of the gpuarray_scan_sharded workspace for a shard of n elements of
 * out_dt (a reduce workspace, room for the gathered totals of up to 4096
 * ranks, and a scan workspace).  Zero-fill once; reusable afterwards. */
size_t gpuarray_scan_sharded_workspace_bytes(ga_dtype_t out_dt, int64_t n);

/* gpuarray_scan over the global array: on rank g,
 *   1. T_g = the fold of the shard with op (one reduce kernel, in out_dt);
 *   2. ncclAllGather of T_0 .. T_{G-1};
 *   3. the local scan of the shard with carry-in c ⊕ T_0 ⊕ ... ⊕ T_{g-1}, c
 *      the fold of carry[0..carry_count) (neutral if none; one more reduce
 *      kernel when carry_count > 0), folded into the scan kernel's tile 0.
 * So out holds elements [start_g, start_g + n) of the scan of the global
 * array (R18: the shard is read twice and written once).  Every
 * argument as gpuarray_scan; widening MAX/MIN scans are GA_ERR_UNSUPPORTED.
 * n may be 0 on some ranks (they still take part in the collective). */
ga_status_t gpuarray_scan_sharded(ga_op_t op, ga_scan_kind_t kind, ga_dtype_t in_dt, ga_dtype_t out_dt, int64_t n,
                                  const void *in, void *out, const void *carry, int64_t carry_count, void *workspace,
                                  size_t workspace_bytes, void *nccl_comm, void *stream);

/* ---- Operator of the CG workload (the paper's
 * "conjugate-gradient-based Krylov solver", applied
 * matrix-free).  Three-point stencil / tridiagonal matvec, dt in {F32, F64}:
 *   y[i] = l*x[i-1] + d_i*x[i] + u*x[i+1],  d_i = diag[i] if diag else d,
 * terms outside [0, n) omitted (Dirichlet boundary), every operation RN left
 * to right, no FMA (R25) — bit-exact against the oracle.  diag is
 * an optional DEVICE array of n elements; y must not overlap x or diag.
 * 1-D Poisson: l = u = -1, d = 2. */
ga_status_t gpuarray_stencil3(ga_dtype_t dt, int64_t n, ga_scalar_t l, ga_scalar_t d, ga_scalar_t u,
                              const void *diag, const void *x, void *y, void *stream);

/* ---- The two fused steps of one CG iteration (NEXT-4).
 * Each is ONE kernel doing what three of the calls above do, with the same
 * per-element rounding, so an iteration is 2 launches and 10 element-sizes of
 * HBM traffic instead of 6 and 14 (R28).  dt in {F32, F64}
 * (others GA_ERR_UNSUPPORTED).  Scalar factors are ga_dscalar_t (device
 * factors read when the kernel runs: graph-capturable).  The workspace is a
 * gpuarray_reduce workspace (gpuarray_reduce_workspace_bytes(dt, n), zeroed
 * once; not shared by calls in flight at the same time).  n == 0 writes 0 to
 * the scalar result.
 *
 * gpuarray_cg_direction:
 *   beta    = RN(beta.scale * RN(*beta.num / *beta.den))  (ga_dscalar_t)
 *   p_out_i = RN(r_i + RN(beta * p_in_i))                  (= gpuarray_axpbyz(1, r, beta, p_in))
 *   ap_i    = (A p_out)_i, A = tridiag(l, d_i, u)          (= gpuarray_stencil3, R25; d_i = diag[i] if diag)
 *   *pap    = sum_i p_out_i * ap_i                          (dot, tolerance R9/R10)
 * r, p_in, diag: n elements, read only; p_out, ap: n elements written; p_out
 * and ap must not overlap each other or any input (neighbours are read);
 * pap: one device element of dt. */
ga_status_t gpuarray_cg_direction(ga_dtype_t dt, int64_t n, ga_dscalar_t beta, const void *r, const void *p_in,
                                  void *p_out, ga_scalar_t l, ga_scalar_t d, ga_scalar_t u, const void *diag, void *ap,
                                  void *pap, void *workspace, size_t workspace_bytes, void *stream);

/* gpuarray_cg_update:
 *   alpha = RN(alpha.scale * RN(*alpha.num / *alpha.den))
 *   x_i  <- RN(x_i + RN(alpha * p_i))                       (= gpuarray_axpbyz_ds(1, x, alpha, p))
 *   r_i  <- RN(r_i + RN(-alpha * ap_i))                     (= gpuarray_axpbyz_ds(1, r, -alpha, ap))
 *   *rr   = sum_i r_i^2 of the updated r                    (norm2sq, tolerance R9/R10)
 * x, r: n elements updated in place; p, ap: n elements read; the four must
 * not overlap; rr: one device element of dt. */
ga_status_t gpuarray_cg_update(ga_dtype_t dt, int64_t n, ga_dscalar_t alpha, void *x, void *r, const void *p,
                               const void *ap, void *rr, void *workspace, size_t workspace_bytes, void *stream);

/* Static strings; never NULL. */
const char *gpuarray_status_string(ga_status_t status);
/* Thread-local detail of the last non-OK status on this thread ("" if none). */
const char *gpuarray_last_error(void);
/* GPUARRAY_ABI_VERSION of the loaded library. */
int gpuarray_abi_version(void);
/* Number of kernels this library has launched in this process (all threads).
 * Evidence for bench.py's "gpu_launches". */
uint64_t gpuarray_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* GPUARRAY_H */
