/* oracle.c — the CPU ORACLE for the GPUArray hot path of arXiv 1304.5553.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1304_5553_b200/) never imports, links or calls it,
 * and shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously correct: ascending-index loops, no blocking, no
 * fusion, no reordering, no intrinsics.  Built with gcc -O2 -ffp-contract=off
 * (no -ffast-math, no -march): every float operation below is one IEEE-754
 * round-to-nearest operation in the type written, with no FMA contraction
 * (reading R1).
 *
 * Passages followed (PAPER.md = /root/reference/PAPER.md):
 *   elementwise  §3.2.4, PAPER.md:449-458  "a statement ... to be executed for
 *                each value of i ... All these instances are required to have
 *                the same length."
 *   map-reduce   §3.2.5, PAPER.md:460-492  result dtype (471-472), map expression
 *                over i (473-477), reduction expression over a,b and a neutral
 *                element (479-485, footnote), scalar result (489-492).
 *   scan         §3.2.6, PAPER.md:496-499  "parallel prefix sums".
 * Readings where the paper is silent (rounding sequence, overflow, neutral
 * elements, NaN, exclusive-scan head, accumulator type) are DESIGN.md R1-R20.
 *
 * Parity pins (tests/test_oracle.py): every function here is pinned against
 * something other than itself — numpy's uncontracted arithmetic, math.fsum,
 * fractions.Fraction brute force, Python big-int arithmetic, closed forms
 * (ramp sums, constant-times-ramp dot, all-ones scan) and SPEC.md worked
 * values; MAX/MIN, including the sign of a zero result (R7), against a
 * Python brute force that orders values by (value, sign) with NaN dropped.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

enum { O_F32 = 0, O_F64 = 1, O_I32 = 2, O_I64 = 3 };
enum { O_SUM = 0, O_MAX = 1, O_MIN = 2 };
enum { O_MAP_ID = 0, O_MAP_MUL = 1, O_MAP_SQUARE = 2 };
enum { O_INCLUSIVE = 0, O_EXCLUSIVE = 1 };

/* maximumNumber / minimumNumber (IEEE 754-2019 §9.6; R6, R7): the
 * larger / smaller operand; a NaN operand loses to a number; -0 is less than
 * +0.  A total order on the non-NaN values, so a fold's result does not
 * depend on the fold order (the GPU folds in tree order). */
static float max_num_f32(float a, float b) {
  if (isnan(a)) return b;
  if (isnan(b)) return a;
  if (a == b) return signbit(a) ? b : a; /* +0 beats -0; equal values are equal */
  return a > b ? a : b;
}
static float min_num_f32(float a, float b) {
  if (isnan(a)) return b;
  if (isnan(b)) return a;
  if (a == b) return signbit(a) ? a : b; /* -0 beats +0 */
  return a < b ? a : b;
}
static double max_num_f64(double a, double b) {
  if (isnan(a)) return b;
  if (isnan(b)) return a;
  if (a == b) return signbit(a) ? b : a;
  return a > b ? a : b;
}
static double min_num_f64(double a, double b) {
  if (isnan(a)) return b;
  if (isnan(b)) return a;
  if (a == b) return signbit(a) ? a : b;
  return a < b ? a : b;
}

/* ------------------------------------------------------------------------ */
/* Elementwise, §3.2.4.  Statement per index i:           */
/*   z[i] = a*x[i] + b*y[i]   read as RN(RN(a*x_i) + RN(b*y_i))   (R1)         */
/*   z[i] = a*x[i] + b        read as RN(RN(a*x_i) + b)                       */
/* Integers wrap modulo 2^w (R4): computed in unsigned arithmetic.            */
/* ------------------------------------------------------------------------ */
void oracle_axpbyz_f32(int64_t n, float a, const float *x, float b, const float *y, float *z) {
  for (int64_t i = 0; i < n; ++i) {
    float ax = a * x[i];
    float by = b * y[i];
    z[i] = ax + by;
  }
}

void oracle_axpbyz_f64(int64_t n, double a, const double *x, double b, const double *y, double *z) {
  for (int64_t i = 0; i < n; ++i) {
    double ax = a * x[i];
    double by = b * y[i];
    z[i] = ax + by;
  }
}

void oracle_axpbyz_i32(int64_t n, int32_t a, const int32_t *x, int32_t b, const int32_t *y, int32_t *z) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t ax = (uint32_t)a * (uint32_t)x[i];
    uint32_t by = (uint32_t)b * (uint32_t)y[i];
    z[i] = (int32_t)(ax + by);
  }
}

void oracle_axpbyz_i64(int64_t n, int64_t a, const int64_t *x, int64_t b, const int64_t *y, int64_t *z) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t ax = (uint64_t)a * (uint64_t)x[i];
    uint64_t by = (uint64_t)b * (uint64_t)y[i];
    z[i] = (int64_t)(ax + by);
  }
}

void oracle_axpbz_f32(int64_t n, float a, const float *x, float b, float *z) {
  for (int64_t i = 0; i < n; ++i) {
    float ax = a * x[i];
    z[i] = ax + b;
  }
}

void oracle_axpbz_f64(int64_t n, double a, const double *x, double b, double *z) {
  for (int64_t i = 0; i < n; ++i) {
    double ax = a * x[i];
    z[i] = ax + b;
  }
}

void oracle_axpbz_i32(int64_t n, int32_t a, const int32_t *x, int32_t b, int32_t *z) {
  for (int64_t i = 0; i < n; ++i) z[i] = (int32_t)((uint32_t)a * (uint32_t)x[i] + (uint32_t)b);
}

void oracle_axpbz_i64(int64_t n, int64_t a, const int64_t *x, int64_t b, int64_t *z) {
  for (int64_t i = 0; i < n; ++i) z[i] = (int64_t)((uint64_t)a * (uint64_t)x[i] + (uint64_t)b);
}

/* ------------------------------------------------------------------------ */
/* Map-reduce SUM over floats, §3.2.5.                     */
/* The tree reduction on the GPU approximates the exact real sum of the       */
/* mapped terms t_i; the oracle computes that sum near-exactly:               */
/*   map: t_i = x_i | x_i*y_i | x_i*x_i, formed   */
/*   exactly in float64 (a product of two fp32 values has <= 48 significant   */
/*   bits).  For fp64 inputs the product p = RN(x*y) and its exact error     */
/*   e = fma(x, y, -p) are both added, so p + e = x*y exactly.               */
/*   reduce "a+b", neutral 0: Neumaier-compensated float64 */
/*   summation in ascending i (BASELINE.json north_star: "reduces in float64  */
/*   with compensated (Kahan) summation").                                    */
/* *sumabs receives sum |t_i| (for the n*2^-24*sum|t_i| tolerance clause).    */
/* ------------------------------------------------------------------------ */
typedef struct { double s, c; } neumaier_t;

static void neumaier_add(neumaier_t *acc, double t) {
  double u = acc->s + t;
  if (fabs(acc->s) >= fabs(t))
    acc->c += (acc->s - u) + t;
  else
    acc->c += (t - u) + acc->s;
  acc->s = u;
}

double oracle_sum_f32(int map, int64_t n, const float *x, const float *y, double *sumabs) {
  neumaier_t acc = {0.0, 0.0};
  neumaier_t abs_acc = {0.0, 0.0};
  for (int64_t i = 0; i < n; ++i) {
    double t;
    if (map == O_MAP_ID) t = (double)x[i];
    else if (map == O_MAP_MUL) t = (double)x[i] * (double)y[i];
    else t = (double)x[i] * (double)x[i];
    neumaier_add(&acc, t);
    neumaier_add(&abs_acc, fabs(t));
  }
  if (sumabs) *sumabs = abs_acc.s + abs_acc.c;
  return acc.s + acc.c;
}

double oracle_sum_f64(int map, int64_t n, const double *x, const double *y, double *sumabs) {
  neumaier_t acc = {0.0, 0.0};
  neumaier_t abs_acc = {0.0, 0.0};
  for (int64_t i = 0; i < n; ++i) {
    if (map == O_MAP_ID) {
      neumaier_add(&acc, x[i]);
      neumaier_add(&abs_acc, fabs(x[i]));
    } else {
      double u = x[i];
      double v = (map == O_MAP_MUL) ? y[i] : x[i];
      double p = u * v;
      double e = fma(u, v, -p);
      neumaier_add(&acc, p);
      neumaier_add(&acc, e);
      neumaier_add(&abs_acc, fabs(p));
    }
  }
  if (sumabs) *sumabs = abs_acc.s + abs_acc.c;
  return acc.s + acc.c;
}

/* ------------------------------------------------------------------------ */
/* Map-reduce SUM over integers: "result dtype" is out_dt. */
/* Inputs are widened to the output width, products and sums wrap modulo     */
/* 2^w_out (R3, R4).  Returned sign-extended in an int64.                     */
/* ------------------------------------------------------------------------ */
static uint64_t load_int(int dt, const void *p, int64_t i) {
  if (dt == O_I32) return (uint64_t)(int64_t)((const int32_t *)p)[i];
  return (uint64_t)((const int64_t *)p)[i];
}

int64_t oracle_sum_int(int map, int in_dt, int out_dt, int64_t n, const void *x, const void *y) {
  uint64_t s = 0;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t u = load_int(in_dt, x, i);
    uint64_t t;
    if (map == O_MAP_ID) t = u;
    else if (map == O_MAP_MUL) t = u * load_int(in_dt, y, i);
    else t = u * u;
    if (out_dt == O_I32) t = (uint64_t)(uint32_t)t;
    s = s + t;
    if (out_dt == O_I32) s = (uint64_t)(uint32_t)s;
  }
  if (out_dt == O_I32) return (int64_t)(int32_t)(uint32_t)s;
  return (int64_t)s;
}

/* ------------------------------------------------------------------------ */
/* Map-reduce MAX / MIN.  Fold from the neutral element:    */
/* MAX: -inf / INT_MIN; MIN: +inf / INT_MAX (R5).  The map is evaluated in    */
/* the input dtype, RN_T(x*y) (R3).  Floats fold with maximumNumber /        */
/* minimumNumber (the non-NaN operand wins, R6; -0 < +0, R7).                 */
/* ------------------------------------------------------------------------ */
double oracle_maxmin_f32(int op, int map, int64_t n, const float *x, const float *y) {
  float acc = (op == O_MAX) ? -INFINITY : INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    float t;
    if (map == O_MAP_ID) t = x[i];
    else if (map == O_MAP_MUL) t = x[i] * y[i];
    else t = x[i] * x[i];
    acc = (op == O_MAX) ? max_num_f32(acc, t) : min_num_f32(acc, t);
  }
  return (double)acc;
}

double oracle_maxmin_f64(int op, int map, int64_t n, const double *x, const double *y) {
  double acc = (op == O_MAX) ? -INFINITY : INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    double t;
    if (map == O_MAP_ID) t = x[i];
    else if (map == O_MAP_MUL) t = x[i] * y[i];
    else t = x[i] * x[i];
    acc = (op == O_MAX) ? max_num_f64(acc, t) : min_num_f64(acc, t);
  }
  return acc;
}

int64_t oracle_maxmin_int(int op, int map, int in_dt, int64_t n, const void *x, const void *y) {
  int64_t acc;
  if (in_dt == O_I32) acc = (op == O_MAX) ? (int64_t)INT32_MIN : (int64_t)INT32_MAX;
  else acc = (op == O_MAX) ? INT64_MIN : INT64_MAX;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t u = load_int(in_dt, x, i);
    uint64_t w;
    if (map == O_MAP_ID) w = u;
    else if (map == O_MAP_MUL) w = u * load_int(in_dt, y, i);
    else w = u * u;
    int64_t t = (in_dt == O_I32) ? (int64_t)(int32_t)(uint32_t)w : (int64_t)w;
    if (op == O_MAX) { if (t > acc) acc = t; }
    else { if (t < acc) acc = t; }
  }
  return acc;
}

/* ------------------------------------------------------------------------ */
/* Scan (prefix sum), §3.2.6, reduction expression "+".    */
/*   inclusive: y_i = c + x_0 + ... + x_i                                     */
/*   exclusive: y_0 = c, y_i = c + x_0 + ... + x_{i-1}   (R13)                */
/* c is the carry-in (0 = the neutral element unless a shard offset is given, */
/* SURVEY.md §8(a) a7).  Running accumulator in the element type; integers   */
/* wrap (R4, R14).  out may alias in.                                          */
/* ------------------------------------------------------------------------ */
void oracle_scan_i32(int kind, int64_t n, const int32_t *in, int32_t *out, int32_t carry) {
  uint32_t acc = (uint32_t)carry;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t v = (uint32_t)in[i];
    if (kind == O_INCLUSIVE) {
      acc = acc + v;
      out[i] = (int32_t)acc;
    } else {
      out[i] = (int32_t)acc;
      acc = acc + v;
    }
  }
}

void oracle_scan_i64(int kind, int64_t n, const int64_t *in, int64_t *out, int64_t carry) {
  uint64_t acc = (uint64_t)carry;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t v = (uint64_t)in[i];
    if (kind == O_INCLUSIVE) {
      acc = acc + v;
      out[i] = (int64_t)acc;
    } else {
      out[i] = (int64_t)acc;
      acc = acc + v;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Scan with the other reduction expressions and element types (§8(f)        */
/* NEXT-2; the paper's scan facility takes a "scan expression" like the      */
/* reduction's, P:496-499 with P:479-485).                                    */
/*   MAX / MIN, any dtype: running fold from the neutral element (or the     */
/*     carry-in), maximumNumber/minimumNumber for floats (R6, R7) — exact.    */
/*   SUM over floats: the exact prefix sums S_i = c + x_0 + ... + x_i,        */
/*     accumulated with Neumaier compensation in float64 and returned as      */
/*     float64 (the GPU's tree/look-back order is an approximation of them;   */
/*     DESIGN.md R22 gives the tolerance).  sumabs_out[i] = |c| + sum|x_j|.   */
/* ------------------------------------------------------------------------ */
void oracle_scan_maxmin_f32(int op, int kind, int64_t n, const float *in, float *out, float carry) {
  float acc = carry;
  for (int64_t i = 0; i < n; ++i) {
    float v = in[i];
    if (kind == O_INCLUSIVE) {
      acc = (op == O_MAX) ? max_num_f32(acc, v) : min_num_f32(acc, v);
      out[i] = acc;
    } else {
      out[i] = acc;
      acc = (op == O_MAX) ? max_num_f32(acc, v) : min_num_f32(acc, v);
    }
  }
}

void oracle_scan_maxmin_f64(int op, int kind, int64_t n, const double *in, double *out, double carry) {
  double acc = carry;
  for (int64_t i = 0; i < n; ++i) {
    double v = in[i];
    if (kind == O_INCLUSIVE) {
      acc = (op == O_MAX) ? max_num_f64(acc, v) : min_num_f64(acc, v);
      out[i] = acc;
    } else {
      out[i] = acc;
      acc = (op == O_MAX) ? max_num_f64(acc, v) : min_num_f64(acc, v);
    }
  }
}

void oracle_scan_maxmin_int(int op, int kind, int dt, int64_t n, const void *in, void *out, int64_t carry) {
  int64_t acc = carry;
  for (int64_t i = 0; i < n; ++i) {
    int64_t v = (dt == O_I32) ? (int64_t)((const int32_t *)in)[i] : ((const int64_t *)in)[i];
    if (kind == O_INCLUSIVE) {
      if (op == O_MAX) { if (v > acc) acc = v; }
      else { if (v < acc) acc = v; }
    }
    if (dt == O_I32) ((int32_t *)out)[i] = (int32_t)acc;
    else ((int64_t *)out)[i] = acc;
    if (kind == O_EXCLUSIVE) {
      if (op == O_MAX) { if (v > acc) acc = v; }
      else { if (v < acc) acc = v; }
    }
  }
}

void oracle_scan_sum_float(int kind, int dt, int64_t n, const void *in, double *out, double carry,
                           double *sumabs_out) {
  neumaier_t acc = {carry, 0.0};
  neumaier_t abs_acc = {fabs(carry), 0.0};
  for (int64_t i = 0; i < n; ++i) {
    double v = (dt == O_F32) ? (double)((const float *)in)[i] : ((const double *)in)[i];
    if (kind == O_INCLUSIVE) {
      neumaier_add(&acc, v);
      neumaier_add(&abs_acc, fabs(v));
    }
    out[i] = acc.s + acc.c;
    if (sumabs_out) sumabs_out[i] = abs_acc.s + abs_acc.c;
    if (kind == O_EXCLUSIVE) {
      neumaier_add(&acc, v);
      neumaier_add(&abs_acc, fabs(v));
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Complex numbers (§8(f) NEXT-3; "seamless support for complex numbers" in  */
/* kernels and GPUArrays).  Arrays are interleaved         */
/* (re, im) pairs of float (c64) or double (c128).                            */
/*   axpbyz: z = a*x + b*y with the complex product written out as           */
/*     re(u*v) = RN(RN(ur*vr) - RN(ui*vi)),  im(u*v) = RN(RN(ur*vi) + RN(ui*vr)) */
/*     and component-wise RN additions (R24), no FMA contraction.             */
/*   sum / dot (x*y) / vdot (conj(x)*y): exact-ish complex sums — each real   */
/*     and imaginary term accumulated separately with Neumaier compensation   */
/*     in float64 (c64 products are exact in float64; c128 products add     */
/*     their fma error terms), returned as (re, im) doubles.                 */
/*   norm2: sum |x_i|^2 = sum (xr^2 + xi^2), a real float64.                  */
/* ------------------------------------------------------------------------ */
enum { O_MAP_CONJ_MUL = 3 };

void oracle_axpbyz_c64(int64_t n, const float *a, const float *x, const float *b, const float *y, float *z) {
  for (int64_t i = 0; i < n; ++i) {
    float xr = x[2 * i], xi = x[2 * i + 1], yr = y[2 * i], yi = y[2 * i + 1];
    float p1 = a[0] * xr, p2 = a[1] * xi, p3 = a[0] * xi, p4 = a[1] * xr;
    float axr = p1 - p2, axi = p3 + p4;
    float q1 = b[0] * yr, q2 = b[1] * yi, q3 = b[0] * yi, q4 = b[1] * yr;
    float byr = q1 - q2, byi = q3 + q4;
    z[2 * i] = axr + byr;
    z[2 * i + 1] = axi + byi;
  }
}

void oracle_axpbyz_c128(int64_t n, const double *a, const double *x, const double *b, const double *y, double *z) {
  for (int64_t i = 0; i < n; ++i) {
    double xr = x[2 * i], xi = x[2 * i + 1], yr = y[2 * i], yi = y[2 * i + 1];
    double p1 = a[0] * xr, p2 = a[1] * xi, p3 = a[0] * xi, p4 = a[1] * xr;
    double axr = p1 - p2, axi = p3 + p4;
    double q1 = b[0] * yr, q2 = b[1] * yi, q3 = b[0] * yi, q4 = b[1] * yr;
    double byr = q1 - q2, byi = q3 + q4;
    z[2 * i] = axr + byr;
    z[2 * i + 1] = axi + byi;
  }
}

/* add u*v (u, v doubles) exactly-ish: the product and, for doubles that are
 * not exact products of floats, its fma error term */
static void neumaier_add_prod(neumaier_t *acc, double u, double v, int exact) {
  double p = u * v;
  neumaier_add(acc, p);
  if (!exact) neumaier_add(acc, fma(u, v, -p));
}

/* map: 0 = ID (sum), 1 = MUL (x*y), 3 = CONJ_MUL (conj(x)*y).  is_c128
 * selects the element type.  out[0], out[1] = (re, im); sumabs[0] = sum of
 * |terms| over both components. */
void oracle_sum_complex(int map, int is_c128, int64_t n, const void *x, const void *y, double *out, double *sumabs) {
  neumaier_t re = {0, 0}, im = {0, 0}, ab = {0, 0};
  const int exact = !is_c128;
  for (int64_t i = 0; i < n; ++i) {
    double xr, xi, yr = 0, yi = 0;
    if (is_c128) {
      xr = ((const double *)x)[2 * i];
      xi = ((const double *)x)[2 * i + 1];
      if (map != O_MAP_ID) { yr = ((const double *)y)[2 * i]; yi = ((const double *)y)[2 * i + 1]; }
    } else {
      xr = ((const float *)x)[2 * i];
      xi = ((const float *)x)[2 * i + 1];
      if (map != O_MAP_ID) { yr = ((const float *)y)[2 * i]; yi = ((const float *)y)[2 * i + 1]; }
    }
    if (map == O_MAP_ID) {
      neumaier_add(&re, xr);
      neumaier_add(&im, xi);
      neumaier_add(&ab, fabs(xr) + fabs(xi));
    } else {
      double s = (map == O_MAP_CONJ_MUL) ? -1.0 : 1.0; /* conj flips the sign of xi */
      neumaier_add_prod(&re, xr, yr, exact);
      neumaier_add_prod(&re, -s * xi, yi, exact);
      neumaier_add_prod(&im, xr, yi, exact);
      neumaier_add_prod(&im, s * xi, yr, exact);
      neumaier_add(&ab, fabs(xr * yr) + fabs(xi * yi) + fabs(xr * yi) + fabs(xi * yr));
    }
  }
  out[0] = re.s + re.c;
  out[1] = im.s + im.c;
  if (sumabs) *sumabs = ab.s + ab.c;
}

double oracle_norm2_complex(int is_c128, int64_t n, const void *x) {
  neumaier_t acc = {0, 0};
  const int exact = !is_c128;
  for (int64_t i = 0; i < n; ++i) {
    double xr = is_c128 ? ((const double *)x)[2 * i] : ((const float *)x)[2 * i];
    double xi = is_c128 ? ((const double *)x)[2 * i + 1] : ((const float *)x)[2 * i + 1];
    neumaier_add_prod(&acc, xr, xr, exact);
    neumaier_add_prod(&acc, xi, xi, exact);
  }
  return acc.s + acc.c;
}

/* ------------------------------------------------------------------------ */
/* Three-point stencil / tridiagonal matvec for the CG workload (§8(f)       */
/* NEXT-4; the paper's Krylov solver, applied matrix-free  */
/* to 1-D Poisson-type systems).  y_i = l*x_{i-1} + d_i*x_i + u*x_{i+1} with */
/* d_i = diag[i] if diag != NULL else d; the terms outside [0, n) are        */
/* omitted (Dirichlet boundary), each operation one RN step, left to right:  */
/*   y_i = RN(RN(RN(l*x_{i-1}) + RN(d_i*x_i)) + RN(u*x_{i+1}))   (R25)       */
/* ------------------------------------------------------------------------ */
void oracle_stencil3_f64(int64_t n, double l, double d, double u, const double *diag, const double *x, double *y) {
  for (int64_t i = 0; i < n; ++i) {
    double di = diag ? diag[i] : d;
    double acc = di * x[i];
    if (i > 0) {
      double t = l * x[i - 1];
      acc = t + acc;
    }
    if (i + 1 < n) {
      double t = u * x[i + 1];
      acc = acc + t;
    }
    y[i] = acc;
  }
}

void oracle_stencil3_f32(int64_t n, float l, float d, float u, const float *diag, const float *x, float *y) {
  for (int64_t i = 0; i < n; ++i) {
    float di = diag ? diag[i] : d;
    float acc = di * x[i];
    if (i > 0) {
      float t = l * x[i - 1];
      acc = t + acc;
    }
    if (i + 1 < n) {
      float t = u * x[i + 1];
      acc = acc + t;
    }
    y[i] = acc;
  }
}

/* ------------------------------------------------------------------------ */
/* GPUArray's other arithmetic operators and cumath-style unary maps        */
/* (§8(f) NEXT-2: GPUArrays "support all arithmetic operators ... many      */
/* special functions are available in pycuda.cumath").    */
/* op: 0 MUL z=x*y, 1 DIV z=x/y, 2 SQRT, 3 ABS, 4 NEG, 5 EXP, 6 LOG,         */
/*     7 SIN, 8 COS, 9 MAX (maxNum), 10 MIN (minNum).                         */
/* IEEE-exact ops (MUL, DIV, SQRT, ABS, NEG, MAX, MIN) are one RN step; the  */
/* transcendental ones are glibc's (R26 gives the ulp bound).       */
/* Integers: MUL (wraps), ABS, NEG (wrap at INT_MIN), MAX, MIN.               */
/* ------------------------------------------------------------------------ */
void oracle_ewmap_f32(int op, int64_t n, const float *x, const float *y, float *z) {
  for (int64_t i = 0; i < n; ++i) {
    float a = x[i], b = y ? y[i] : 0.0f, r = 0.0f;
    switch (op) {
      case 0: r = a * b; break;
      case 1: r = a / b; break;
      case 2: r = sqrtf(a); break;
      case 3: r = fabsf(a); break;
      case 4: r = -a; break;
      case 5: r = expf(a); break;
      case 6: r = logf(a); break;
      case 7: r = sinf(a); break;
      case 8: r = cosf(a); break;
      case 9: r = max_num_f32(a, b); break;
      case 10: r = min_num_f32(a, b); break;
    }
    z[i] = r;
  }
}

void oracle_ewmap_f64(int op, int64_t n, const double *x, const double *y, double *z) {
  for (int64_t i = 0; i < n; ++i) {
    double a = x[i], b = y ? y[i] : 0.0, r = 0.0;
    switch (op) {
      case 0: r = a * b; break;
      case 1: r = a / b; break;
      case 2: r = sqrt(a); break;
      case 3: r = fabs(a); break;
      case 4: r = -a; break;
      case 5: r = exp(a); break;
      case 6: r = log(a); break;
      case 7: r = sin(a); break;
      case 8: r = cos(a); break;
      case 9: r = max_num_f64(a, b); break;
      case 10: r = min_num_f64(a, b); break;
    }
    z[i] = r;
  }
}

void oracle_ewmap_int(int op, int dt, int64_t n, const void *x, const void *y, void *z) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = load_int(dt, x, i), b = y ? (int64_t)load_int(dt, y, i) : 0, r = 0;
    uint64_t ua = (uint64_t)a;
    switch (op) {
      case 0: r = (int64_t)(ua * (uint64_t)b); break;
      case 3: r = a < 0 ? (int64_t)(0 - ua) : a; break;
      case 4: r = (int64_t)(0 - ua); break;
      case 9: r = a > b ? a : b; break;
      case 10: r = a < b ? a : b; break;
    }
    if (dt == O_I32) ((int32_t *)z)[i] = (int32_t)(uint32_t)(uint64_t)r;
    else ((int64_t *)z)[i] = r;
  }
}
