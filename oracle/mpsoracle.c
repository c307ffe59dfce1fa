/*
 * mpsoracle.c -- TEST INFRASTRUCTURE ONLY (the CPU checker, never the product).
 *
 * Plain-C restatement of the reference's multi-component arithmetic, CSR SpMV
 * (both accumulation orders), fused complex SpMV and conjugate gradient.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/mps/).
 *
 * Parity pin: this restatement is checked bit-for-bit against the reference
 * itself (oracle/_ref/libmpsref.so, compiled from the reference headers by
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 *
 * Build: gcc -O2 -ffp-contract=off (the reference's only global flag,
 * proj/CMakeLists.txt:14): no FMA contraction, fma() only where the
 * reference calls std::fma.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ---------------------------------------------------------------- EFTs ---
 * eft.hpp:26-30 quick_two_sum_raw, :34-41 two_sum, :53-59 two_prod_fma,
 * :63-71 three_sum, :74-80 three_sum2. */
static inline void qts(double a, double b, double *s, double *e) {
  double ss = a + b;
  *e = b - (ss - a);
  *s = ss;
}
static inline void two_sum(double a, double b, double *s, double *e) {
  double ss = a + b;
  double v = ss - a;
  *e = (a - (ss - v)) + (b - v);
  *s = ss;
}
static inline void two_prod(double a, double b, double *p, double *e) {
  double pp = a * b;
  *e = fma(a, b, -pp);
  *p = pp;
}
static inline void three_sum(double *a, double *b, double *c) {
  double t1, t2, s1, t3, s2, s3;
  two_sum(*a, *b, &t1, &t2);
  two_sum(*c, t1, &s1, &t3);
  two_sum(t2, t3, &s2, &s3);
  *a = s1;
  *b = s2;
  *c = s3;
}
static inline void three_sum2(double *a, double *b, double c) {
  double t1, t2, s1, t3;
  two_sum(*a, *b, &t1, &t2);
  two_sum(c, t1, &s1, &t3);
  *a = s1;
  *b = t2 + t3;
}

/* ------------------------------------------------------------ renorm_n ---
 * multicomp.hpp:43-78.  Non-finite lead: plain left fold from +0 into c0.
 * Backward Dekker sweep, then forward collect emitting a component whenever
 * the low part is nonzero; the last slot absorbs the rest with plain adds. */
static void renorm_n(int K, int N, const double *tin, double *r) {
  double t[5] = {0, 0, 0, 0, 0};
  for (int i = 0; i < N; ++i) t[i] = tin[i];
  for (int i = 0; i < K; ++i) r[i] = 0.0;
  if (!isfinite(t[0])) {
    double s = 0.0;
    for (int i = 0; i < N; ++i) s += t[i];
    r[0] = s;
    return;
  }
  double s = t[N - 1];
  for (int i = N - 1; i-- > 0;) {
    double hi, lo;
    qts(t[i], s, &hi, &lo);
    s = hi;
    t[i + 1] = lo;
  }
  t[0] = s;
  int k = 0;
  s = t[0];
  for (int i = 1; i < N; ++i) {
    if (k == K - 1) {
      s += t[i];
      continue;
    }
    double hi, lo;
    qts(s, t[i], &hi, &lo);
    if (lo != 0.0) {
      r[k++] = hi;
      s = lo;
    } else {
      s = hi;
    }
  }
  r[k] = s;
}

/* ------------------------------------------------------------ DD cores ---
 * multicomp.hpp:80-110 */
static void dd_add(const double *x, const double *y, double *r) {
  double s, e, w;
  two_sum(x[0], y[0], &s, &e);
  w = x[1] + y[1];
  e = e + w;
  qts(s, e, &r[0], &r[1]);
}
static void dd_mul(const double *x, const double *y, double *r) {
  double p1, p2, w1, w2, w3;
  two_prod(x[0], y[0], &p1, &p2);
  w1 = x[0] * y[1];
  w2 = x[1] * y[0];
  w3 = w1 + w2;
  p2 = p2 + w3;
  qts(p1, p2, &r[0], &r[1]);
}
static void dd_mul_d(const double *x, double y, double *r) {
  double p1, p2;
  two_prod(x[0], y, &p1, &p2);
  p2 = fma(x[1], y, p2);
  qts(p1, p2, &r[0], &r[1]);
}

/* ----------------------------------------------------- QD/TD prenorms ---
 * multicomp.hpp:112-215 */
static void qd_add_prenorm(const double *x, const double *y, double *out) {
  double s0, t0, s1, t1, s2, t2, s3, t3;
  two_sum(x[0], y[0], &s0, &t0);
  two_sum(x[1], y[1], &s1, &t1);
  two_sum(x[2], y[2], &s2, &t2);
  two_sum(x[3], y[3], &s3, &t3);
  double s1b, t0b;
  two_sum(s1, t0, &s1b, &t0b);
  s1 = s1b;
  t0 = t0b;
  three_sum(&s2, &t0, &t1);
  three_sum2(&s3, &t0, t2);
  t0 = t0 + t1 + t3;
  out[0] = s0;
  out[1] = s1;
  out[2] = s2;
  out[3] = s3;
  out[4] = t0;
}
static void qd_mul_prenorm(const double *a, const double *b, double *out) {
  double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5;
  two_prod(a[0], b[0], &p0, &q0);
  two_prod(a[0], b[1], &p1, &q1);
  two_prod(a[1], b[0], &p2, &q2);
  two_prod(a[0], b[2], &p3, &q3);
  two_prod(a[1], b[1], &p4, &q4);
  two_prod(a[2], b[0], &p5, &q5);
  three_sum(&p1, &p2, &q0);
  three_sum(&p2, &q1, &q2);
  three_sum(&p3, &p4, &p5);
  double s0, t0, s1, t1, s2;
  two_sum(p2, p3, &s0, &t0);
  two_sum(q1, p4, &s1, &t1);
  s2 = q2 + p5;
  double s1b, t0b;
  two_sum(s1, t0, &s1b, &t0b);
  s1 = s1b;
  s2 = s2 + (t0b + t1);
  /* multicomp.hpp:156, strictly left to right, separate multiplies */
  s1 = s1 + (a[0] * b[3] + a[1] * b[2] + a[2] * b[1] + a[3] * b[0] + q0 + q3 + q4 + q5);
  out[0] = p0;
  out[1] = p1;
  out[2] = s0;
  out[3] = s1;
  out[4] = s2;
}
static void qd_mul_d_prenorm(const double *a, double b, double *out) {
  double p0, q0, p1, q1, p2, q2, p3;
  two_prod(a[0], b, &p0, &q0);
  two_prod(a[1], b, &p1, &q1);
  two_prod(a[2], b, &p2, &q2);
  p3 = a[3] * b;
  double s1, s2;
  two_sum(q0, p1, &s1, &s2);
  three_sum(&s2, &q1, &p2);
  three_sum2(&q1, &p2, p3);
  double s3 = q1;
  double s4 = q2 + p2;
  out[0] = p0;
  out[1] = s1;
  out[2] = s2;
  out[3] = s3;
  out[4] = s4;
}
static void td_mul_d_prenorm(const double *a, double b, double *out) {
  double p0, q0, p1, q1, p2, q2;
  two_prod(a[0], b, &p0, &q0);
  two_prod(a[1], b, &p1, &q1);
  two_prod(a[2], b, &p2, &q2);
  double s1, s2;
  two_sum(q0, p1, &s1, &s2);
  three_sum(&s2, &q1, &p2);
  double s3 = q2 + p2;
  out[0] = p0;
  out[1] = s1;
  out[2] = s2;
  out[3] = s3;
}

/* ------------------------------------------------ public MC operations ---
 * multicomp.hpp:225-277 (add/mul/mul_by_double), :279-289 (negate/sub). */
ORC_API void orc_add(int K, const double *x, const double *y, double *r) {
  double t[5];
  if (K == 2) {
    dd_add(x, y, r);
  } else if (K == 3) {
    double xe[4] = {x[0], x[1], x[2], 0.0}, ye[4] = {y[0], y[1], y[2], 0.0};
    qd_add_prenorm(xe, ye, t);
    renorm_n(3, 5, t, r);
  } else {
    qd_add_prenorm(x, y, t);
    renorm_n(4, 5, t, r);
  }
}
ORC_API void orc_mul(int K, const double *x, const double *y, double *r) {
  double t[5];
  if (K == 2) {
    dd_mul(x, y, r);
  } else if (K == 3) {
    double xe[4] = {x[0], x[1], x[2], 0.0}, ye[4] = {y[0], y[1], y[2], 0.0};
    qd_mul_prenorm(xe, ye, t);
    renorm_n(3, 5, t, r);
  } else {
    qd_mul_prenorm(x, y, t);
    renorm_n(4, 5, t, r);
  }
}
ORC_API void orc_mul_d(int K, const double *x, double y, double *r) {
  double t[5];
  if (K == 2) {
    dd_mul_d(x, y, r);
  } else if (K == 3) {
    td_mul_d_prenorm(x, y, t);
    renorm_n(3, 4, t, r);
  } else {
    qd_mul_d_prenorm(x, y, t);
    renorm_n(4, 5, t, r);
  }
}
ORC_API void orc_sub(int K, const double *x, const double *y, double *r) {
  double ny[4];
  for (int i = 0; i < K; ++i) ny[i] = -y[i];
  orc_add(K, x, ny, r);
}
/* multicomp.hpp:291-302 long division */
ORC_API void orc_div(int K, const double *a, const double *b, double *out) {
  double q[5], r[4], t[4];
  for (int i = 0; i < K; ++i) r[i] = a[i];
  for (int i = 0; i <= K; ++i) {
    q[i] = r[0] / b[0];
    if (i < K) {
      orc_mul_d(K, b, q[i], t);
      orc_sub(K, r, t, r);
    }
  }
  renorm_n(K, K + 1, q, out);
}
/* multicomp.hpp:304-322 Newton on 1/sqrt(a) */
ORC_API void orc_sqrt(int K, const double *a, double *out) {
  for (int i = 0; i < K; ++i) out[i] = 0.0;
  if (a[0] == 0.0) return;
  if (a[0] < 0.0 || isnan(a[0])) {
    out[0] = NAN;
    return;
  }
  double x[4] = {0, 0, 0, 0}, one[4] = {1.0, 0, 0, 0}, xx[4], axx[4], e[4], xe[4], h[4];
  x[0] = 1.0 / sqrt(a[0]);
  int iters = (K == 4) ? 3 : 2;
  for (int i = 0; i < iters; ++i) {
    orc_mul(K, x, x, xx);
    orc_mul(K, a, xx, axx);
    orc_sub(K, one, axx, e);
    orc_mul(K, x, e, xe);
    orc_mul_d(K, xe, 0.5, h);
    orc_add(K, x, h, x);
  }
  double r[4], rr[4], d[4], dx[4];
  orc_mul(K, a, x, r);
  orc_mul(K, r, r, rr);
  orc_sub(K, a, rr, d);
  orc_mul(K, d, x, dx);
  orc_mul_d(K, dx, 0.5, h);
  orc_add(K, r, h, out);
}
/* multicomp.hpp:329-335 */
ORC_API double orc_to_double(int K, const double *x) {
  double s = x[K - 1];
  for (int i = K - 2; i >= 0; --i) s = x[i] + s;
  return s;
}
/* multicomp.hpp:342-351 */
ORC_API int orc_compare(int K, const double *x, const double *y) {
  if (isnan(x[0]) || isnan(y[0])) return -2;
  for (int i = 0; i < K; ++i) {
    if (x[i] < y[i]) return -1;
    if (x[i] > y[i]) return 1;
  }
  return 0;
}

/* --------------------------------------------------------------- SpMV ---
 * Row accumulation in the reference's two orders.
 * SCALAR (lanes off): kernels.hpp:90-99 row_sum_scalar.
 * LANE4  (lanes on) : kernels.hpp:103-121 row_sum_lanes_pure; the 4-lane
 *   batch ops are bit-identical per lane to the scalar ops
 *   (lanebatch.hpp:79-89), so each lane is a scalar chain.
 * Pure mode product: mul(a, v), matrix operand first (kernels.hpp:52-54).
 * Mixed mode product: mul_by_double(v, a) (kernels.hpp:55-58, :123-142). */
static void row_sum(int K, int lanes, int mixed, int64_t b, int64_t e, const int64_t *indices,
                    const double *vals, int64_t nnz, const double *x, double *out) {
  double acc[4] = {0, 0, 0, 0}, a[4], p[4];
#define LOAD_A(k)                                                      \
  do {                                                                 \
    if (!mixed)                                                        \
      for (int j = 0; j < K; ++j) a[j] = vals[(int64_t)j * nnz + (k)]; \
  } while (0)
#define PROD(k)                                                        \
  do {                                                                 \
    const double *xv = x + indices[(k)] * K;                           \
    if (mixed)                                                         \
      orc_mul_d(K, xv, vals[(k)], p);                                  \
    else {                                                             \
      LOAD_A(k);                                                       \
      orc_mul(K, a, xv, p);                                            \
    }                                                                  \
  } while (0)
  if (!lanes) {
    for (int64_t k = b; k < e; ++k) {
      PROD(k);
      orc_add(K, acc, p, acc);
    }
  } else {
    double L[4][4];
    memset(L, 0, sizeof(L));
    int64_t k = b;
    for (; k + 4 <= e; k += 4) {
      for (int l = 0; l < 4; ++l) {
        PROD(k + l);
        orc_add(K, L[l], p, L[l]);
      }
    }
    /* s = ((zero + L0) + L1) + L2; s = s + L3  (kernels.hpp:114-115) */
    for (int l = 0; l < 4; ++l) orc_add(K, acc, L[l], acc);
    for (; k < e; ++k) {
      PROD(k);
      orc_add(K, acc, p, acc);
    }
  }
#undef PROD
#undef LOAD_A
  for (int j = 0; j < K; ++j) out[j] = acc[j];
}

/* kernels.hpp:348-366 (spmv).  The row partition does not change results
 * (kernels.hpp:20-29), so this runs rows in order on one thread.
 * vals: K component planes [K][nnz] (CsrValues SoA, sparse.hpp:47-67),
 * or one binary64 plane when mixed != 0. x, y: AoS [n][K]. Returns 0, or -1
 * on dimension mismatch (the reference throws std::invalid_argument). */
ORC_API int orc_spmv(int K, int lanes, int mixed, int64_t nrows, int64_t ncols, int64_t xlen,
                     const int64_t *indptr, const int64_t *indices, const double *vals,
                     const double *x, double *y) {
  if (xlen != ncols) return -1;
  int64_t nnz = indptr[nrows];
  for (int64_t i = 0; i < nrows; ++i)
    row_sum(K, lanes, mixed, indptr[i], indptr[i + 1], indices, vals, nnz, x, y + i * K);
  return 0;
}

/* kernels.hpp:399-416: four real products then y.re = rr - ii (sub =
 * add(x, negate(y)), multicomp.hpp:286-289), y.im = ri + ir. re and im share
 * one structure here (check_split_structure, sparse.hpp:254-259). */
ORC_API int orc_spmv_complex(int K, int lanes, int mixed, int64_t nrows, int64_t ncols, int64_t xlen,
                             const int64_t *indptr, const int64_t *indices, const double *vre,
                             const double *vim, const double *xre, const double *xim, double *yre,
                             double *yim) {
  if (xlen != ncols) return -1;
  int64_t nnz = indptr[nrows];
  for (int64_t i = 0; i < nrows; ++i) {
    double rr[4], ii[4], ri[4], ir[4];
    row_sum(K, lanes, mixed, indptr[i], indptr[i + 1], indices, vre, nnz, xre, rr);
    row_sum(K, lanes, mixed, indptr[i], indptr[i + 1], indices, vim, nnz, xim, ii);
    row_sum(K, lanes, mixed, indptr[i], indptr[i + 1], indices, vre, nnz, xim, ri);
    row_sum(K, lanes, mixed, indptr[i], indptr[i + 1], indices, vim, nnz, xre, ir);
    orc_sub(K, rr, ii, yre + i * K);
    orc_add(K, ri, ir, yim + i * K);
  }
  return 0;
}

/* ------------------------------------------------------------- SpTMV ---
 * kernels.hpp:368-394 (sptmv): with one thread, one accumulator y (all +0)
 * updated row by row, y[col_k] = y[col_k] + mul_term(a_k, v_i), i ascending
 * (sptmv_block :214-225; the lane variant SptRow :227-322 performs the same
 * per-element ops, so lanes do not change the bits).  With T > 1 threads:
 * partition_rows(T) blocks (:63-80), one zero accumulator per block, merged
 * in thread order y = acc_0; y[j] = y[j] + acc_t[j] (:386-392). */
static void sptmv_block(int K, int mixed, int64_t r0, int64_t r1, const int64_t *indptr,
                        const int64_t *indices, const double *vals, int64_t nnz, const double *v,
                        double *acc) {
  double a[4], p[4];
  for (int64_t i = r0; i < r1; ++i) {
    const double *vi = v + i * K;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
      double *yj = acc + indices[k] * K;
      if (mixed) {
        orc_mul_d(K, vi, vals[k], p);
      } else {
        for (int j = 0; j < K; ++j) a[j] = vals[(int64_t)j * nnz + k];
        orc_mul(K, a, vi, p);
      }
      orc_add(K, yj, p, yj);
    }
  }
}
static int64_t lower_bound_i64(const int64_t *a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
ORC_API int orc_sptmv(int K, int mixed, int threads, int64_t nrows, int64_t ncols, int64_t vlen,
                      const int64_t *indptr, const int64_t *indices, const double *vals,
                      const double *v, double *y) {
  if (vlen != nrows) return -1;
  int64_t nnz = indptr[nrows];
  if (threads < 1) threads = 1;
  memset(y, 0, sizeof(double) * (size_t)(ncols * K));
  if (threads == 1 || nrows == 0) {
    sptmv_block(K, mixed, 0, nrows, indptr, indices, vals, nnz, v, y);
    return 0;
  }
  double *acc = (double *)malloc(sizeof(double) * (size_t)(ncols * K) + 8);
  int64_t b0 = 0;
  for (int t = 0; t < threads; ++t) {
    /* partition_rows: bounds[t] = lower_bound(indptr, total*t/parts) */
    int64_t b1 = (t + 1 == threads) ? nrows : lower_bound_i64(indptr, nrows, nnz * (t + 1) / threads);
    if (b1 < b0) b1 = b0;
    double *dst = (t == 0) ? y : acc;
    if (t > 0) memset(acc, 0, sizeof(double) * (size_t)(ncols * K));
    sptmv_block(K, mixed, b0, b1, indptr, indices, vals, nnz, v, dst);
    if (t > 0)
      for (int64_t j = 0; j < ncols; ++j) orc_add(K, y + j * K, acc + j * K, y + j * K);
    b0 = b1;
  }
  free(acc);
  return 0;
}
/* kernels.hpp:419-441: four real transposed products, then rr - ii / ri + ir,
 * or with conjugate (the adjoint) rr + ii / ri - ir. */
ORC_API int orc_sptmv_complex(int K, int mixed, int threads, int conj, int64_t nrows, int64_t ncols,
                              int64_t vlen, const int64_t *indptr, const int64_t *indices,
                              const double *vre, const double *vim, const double *xre, const double *xim,
                              double *yre, double *yim) {
  if (vlen != nrows) return -1;
  size_t nb = sizeof(double) * (size_t)(ncols * K) + 8;
  double *rr = malloc(nb), *ii = malloc(nb), *ri = malloc(nb), *ir = malloc(nb);
  orc_sptmv(K, mixed, threads, nrows, ncols, vlen, indptr, indices, vre, xre, rr);
  orc_sptmv(K, mixed, threads, nrows, ncols, vlen, indptr, indices, vim, xim, ii);
  orc_sptmv(K, mixed, threads, nrows, ncols, vlen, indptr, indices, vre, xim, ri);
  orc_sptmv(K, mixed, threads, nrows, ncols, vlen, indptr, indices, vim, xre, ir);
  for (int64_t j = 0; j < ncols; ++j) {
    if (conj) {
      orc_add(K, rr + j * K, ii + j * K, yre + j * K);
      orc_sub(K, ri + j * K, ir + j * K, yim + j * K);
    } else {
      orc_sub(K, rr + j * K, ii + j * K, yre + j * K);
      orc_add(K, ri + j * K, ir + j * K, yim + j * K);
    }
  }
  free(rr); free(ii); free(ri); free(ir);
  return 0;
}

/* ----------------------------------------------------------- checksum ---
 * bench.hpp:113-150: FNV-1a 64 over the 8 little-endian bytes of every
 * component, elements in order, components j = 0..K-1. */
ORC_API uint64_t orc_checksum(int K, int64_t n, const double *v) {
  uint64_t h = 14695981039346656037ull;
  for (int64_t i = 0; i < n * K; ++i) {
    uint64_t bits;
    memcpy(&bits, &v[i], 8);
    for (int b = 0; b < 8; ++b) {
      h ^= (bits >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}
ORC_API uint64_t orc_checksum_complex(int K, int64_t n, const double *re, const double *im) {
  return orc_checksum(K, n, re) * 1099511628211ull ^ orc_checksum(K, n, im);
}

/* ---------------------------------------------------- bound helpers ---
 * Checker support for the fast-mode componentwise bound
 * |y_gpu - y_ref| <= 4 * rowlen * u * sum_j |a_ij| |x_j|  (BASELINE.json).
 * orc_exact_diff returns |a - b| for two K-component values: the 2K terms are
 * summed error-free into a nonoverlapping expansion (Shewchuk grow-expansion)
 * and the expansion is then rounded once. */
ORC_API double orc_exact_diff(int K, const double *a, const double *b) {
  double e[16];
  int m = 0;
  for (int t = 0; t < 2 * K; ++t) {
    double q = t < K ? a[t] : -b[t - K];
    if (!isfinite(q)) return (a[0] == b[0]) ? 0.0 : INFINITY;
    for (int i = 0; i < m; ++i) {
      double s, err;
      two_sum(q, e[i], &s, &err);
      e[i] = err;
      q = s;
    }
    e[m++] = q;
  }
  /* e is ordered by increasing magnitude; fold small to large */
  double s = 0.0;
  for (int i = 0; i < m; ++i) s += e[i];
  return fabs(s);
}

/* orc_exact_diff over n AoS rows (the full-size bound checks). */
ORC_API void orc_exact_diff_vec(int K, int64_t n, const double *a, const double *b, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_exact_diff(K, a + i * K, b + i * K);
}

/* Per-row sum_j |a_ij| |x_j| on leading components, and row lengths.
 * For complex, the caller passes the re/im planes and sums all four. */
ORC_API void orc_abs_rowsum(int K, int64_t nrows, const int64_t *indptr, const int64_t *indices,
                            const double *lead_vals, const double *x, double *out) {
  for (int64_t i = 0; i < nrows; ++i) {
    double s = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
      s += fabs(lead_vals[k]) * fabs(x[indices[k] * K]);
    out[i] = s;
  }
}

/* ------------------------------------------------------------------ CG ---
 * krylov.hpp:238-281 solve_cg with solver_init :160-201, record_step
 * :203-213, close_report :215-224, finish_true_residual :226-232.
 * dot :122-128 (sequential acc = acc + u*v), norm2 :130-134, axpy :136-140
 * (y = y + alpha*x).  Status codes follow SolverStatus (krylov.hpp:46):
 * 0 converged, 1 max_iterations, 2 breakdown, 3 diverged. */
static void vdot(int K, int64_t n, const double *u, const double *v, double *acc) {
  double p[4];
  for (int j = 0; j < K; ++j) acc[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    orc_mul(K, u + i * K, v + i * K, p);
    orc_add(K, acc, p, acc);
  }
}

ORC_API int orc_cg(int K, int lanes, int64_t n, const int64_t *indptr, const int64_t *indices,
                   const double *vals, const double *b, double rel_tol, double abs_tol,
                   int64_t max_iters, double *x, double *history, int64_t *iterations,
                   int *status, double *rhs_norm, double *final_true_residual) {
  if (!(rel_tol > 0.0) || !(abs_tol > 0.0) || max_iters < 1) return -1;
  size_t bytes = (size_t)n * K * sizeof(double);
  double *r = malloc(bytes), *p = malloc(bytes), *q = malloc(bytes);
  double t[4], bn[4], thr[4], tmp[4], rho[4], sigma[4], alpha[4], malpha[4], rho_next[4],
      rnorm[4], beta[4];
  int64_t nh = 0;
  for (int64_t i = 0; i < n * K; ++i) x[i] = 0.0;
  memcpy(r, b, bytes);
  /* solver_init: threshold = bnorm*rel_tol + abs_tol (krylov.hpp:185-186) */
  vdot(K, n, b, b, t);
  orc_sqrt(K, t, bn);
  orc_mul_d(K, bn, rel_tol, tmp);
  double at[4] = {abs_tol, 0, 0, 0};
  orc_add(K, tmp, at, thr);
  *rhs_norm = orc_to_double(K, bn);
  double divergence_cap = 1e6 * *rhs_norm + 1e6 * abs_tol;
  double breakdown_floor = 1e-3 * abs_tol;
  vdot(K, n, r, r, t);
  orc_sqrt(K, t, rnorm);
  history[nh++] = orc_to_double(K, rnorm);
  int st = 1;
  int64_t k = 0;
  int c = orc_compare(K, rnorm, thr);
  if (c == 0 || c == -1) {
    st = 0;
  } else {
    memcpy(p, r, bytes);
    vdot(K, n, r, r, rho);
    for (k = 1; k <= max_iters; ++k) {
      orc_spmv(K, lanes, 0, n, n, n, indptr, indices, vals, p, q);
      vdot(K, n, p, q, sigma);
      double sd = orc_to_double(K, sigma);
      if (!isfinite(sd) || fabs(sd) < breakdown_floor) {
        st = 2;
        k = k - 1;
        break;
      }
      orc_div(K, rho, sigma, alpha);
      for (int j = 0; j < K; ++j) malpha[j] = -alpha[j];
      for (int64_t i = 0; i < n; ++i) {
        orc_mul(K, alpha, p + i * K, tmp);
        orc_add(K, x + i * K, tmp, x + i * K);
      }
      for (int64_t i = 0; i < n; ++i) {
        orc_mul(K, malpha, q + i * K, tmp);
        orc_add(K, r + i * K, tmp, r + i * K);
      }
      vdot(K, n, r, r, rho_next);
      orc_sqrt(K, rho_next, rnorm);
      double rd = orc_to_double(K, rnorm);
      history[nh++] = rd;
      if (!isfinite(rd)) {
        st = 2;
        break;
      }
      c = orc_compare(K, rnorm, thr);
      if (c == 0 || c == -1) {
        st = 0;
        break;
      }
      if (rd > divergence_cap) {
        st = 3;
        break;
      }
      orc_div(K, rho_next, rho, beta);
      for (int64_t i = 0; i < n; ++i) {
        orc_mul(K, beta, p + i * K, tmp);
        orc_add(K, r + i * K, tmp, p + i * K);
      }
      memcpy(rho, rho_next, sizeof(rho));
    }
    if (k > max_iters) k = max_iters;
  }
  *iterations = k;
  *status = st;
  /* finish_true_residual: ||b - A x|| from a fresh product */
  orc_spmv(K, lanes, 0, n, n, n, indptr, indices, vals, x, q);
  for (int64_t i = 0; i < n; ++i) orc_sub(K, b + i * K, q + i * K, q + i * K);
  vdot(K, n, q, q, t);
  orc_sqrt(K, t, tmp);
  *final_true_residual = orc_to_double(K, tmp);
  free(r);
  free(p);
  free(q);
  return (int)nh;
}

/* ------------------------------------------------------ Krylov solvers ---
 * krylov.hpp:238-594 -- solve_cg, solve_bicg, solve_cgs, solve_bicgstab,
 * solve_gpbicg, dispatched on `method` like solve() :596-606 (KrylovMethod
 * order, krylov.hpp:24).  Common parts: solver_init :160-201 (x0 :174-181),
 * record_step :203-213, close_report :215-224, finish_true_residual
 * :226-232, tiny :234.  The operator is CsrOperator (krylov.hpp:101-120):
 * apply = spmv in the lanes order, apply_transposed = sptmv at `threads`.
 * reason codes (the SolverReport detail text after "<method>: "):
 *   1 "<p, Ap> vanished"  2 "non-finite residual"  3 "<r~, r> vanished"
 *   4 "<p~, Ap> vanished" 5 "<r~, Ap> vanished"    6 "<t, t> vanished"
 *   7 "omega vanished"    8 "<At, At> vanished"    9 "zeta/eta system is singular"
 *  10 "zeta vanished" */
typedef struct {
  int K, lanes, threads;
  int64_t n;
  const int64_t *indptr, *indices;
  const double *vals;
  double thr[4], cap, floor;
  double *hist;
  int64_t nh;
  int mixed; /* CsrOperator<double> with K-component vectors (bench.cpp:550-557) */
} KrCtx;

static void kr_apply(const KrCtx *c, const double *x, double *y) {
  orc_spmv(c->K, c->lanes, c->mixed, c->n, c->n, c->n, c->indptr, c->indices, c->vals, x, y);
}
static void kr_apply_t(const KrCtx *c, const double *x, double *y) {
  orc_sptmv(c->K, c->mixed, c->threads, c->n, c->n, c->n, c->indptr, c->indices, c->vals, x, y);
}
static void kr_axpy(int K, int64_t n, const double *alpha, const double *x, double *y) {
  double t[4];
  for (int64_t i = 0; i < n; ++i) {
    orc_mul(K, alpha, x + i * K, t);
    orc_add(K, y + i * K, t, y + i * K);
  }
}
static void kr_norm2(int K, int64_t n, const double *v, double *out) {
  double d[4];
  vdot(K, n, v, v, d);
  orc_sqrt(K, d, out);
}
static void kr_neg(int K, const double *a, double *r) {
  for (int j = 0; j < K; ++j) r[j] = -a[j];
}
static int kr_tiny(double v, double floor) { return !isfinite(v) || fabs(v) < floor; }
static int kr_le(int K, const double *a, const double *b) {
  int c = orc_compare(K, a, b);
  return c == 0 || c == -1;
}
/* record_step: 0 continue, 1 converged, 2 diverged, 3 non-finite */
static int kr_record(KrCtx *c, const double *rnorm) {
  double rd = orc_to_double(c->K, rnorm);
  c->hist[c->nh++] = rd;
  if (!isfinite(rd)) return 3;
  if (kr_le(c->K, rnorm, c->thr)) return 1;
  if (rd > c->cap) return 2;
  return 0;
}
/* step -> (status, reason) as close_report is called after a stop */
static void kr_stop(int step, int *status, int *reason) {
  *status = step == 1 ? 0 : step == 2 ? 3 : 2;
  *reason = step == 3 ? 2 : 0;
}

#define KR_VEC(name) double *name = (double *)calloc((size_t)(n * K) + 1, sizeof(double))
#define KR_BREAK(why, it) \
  do {                    \
    *status = 2;          \
    *reason = (why);      \
    *iters = (it);        \
    goto out;             \
  } while (0)
#define KR_RECORD(rn)                     \
  do {                                    \
    int step_ = kr_record(c, (rn));       \
    if (step_) {                          \
      kr_stop(step_, status, reason);     \
      *iters = k;                         \
      goto out;                           \
    }                                     \
  } while (0)

static void kr_cg(KrCtx *c, double *x, double *r, int64_t max_iters, int64_t *iters, int *status,
                  int *reason) {
  const int K = c->K;
  const int64_t n = c->n;
  KR_VEC(p);
  KR_VEC(q);
  double rho[4], sigma[4], alpha[4], ma[4], rn[4], rho_next[4], beta[4], t[4];
  int64_t k;
  memcpy(p, r, sizeof(double) * (size_t)(n * K));
  vdot(K, n, r, r, rho);
  for (k = 1; k <= max_iters; ++k) {
    kr_apply(c, p, q);
    vdot(K, n, p, q, sigma);
    if (kr_tiny(orc_to_double(K, sigma), c->floor)) KR_BREAK(1, k - 1);
    orc_div(K, rho, sigma, alpha);
    kr_neg(K, alpha, ma);
    kr_axpy(K, n, alpha, p, x);
    kr_axpy(K, n, ma, q, r);
    vdot(K, n, r, r, rho_next);
    orc_sqrt(K, rho_next, rn);
    KR_RECORD(rn);
    orc_div(K, rho_next, rho, beta);
    for (int64_t i = 0; i < n; ++i) {
      orc_mul(K, beta, p + i * K, t);
      orc_add(K, r + i * K, t, p + i * K);
    }
    memcpy(rho, rho_next, sizeof(rho));
  }
  *status = 1;
  *iters = max_iters;
out:
  free(p);
  free(q);
}

static void kr_bicg(KrCtx *c, double *x, double *r, int64_t max_iters, int64_t *iters, int *status,
                    int *reason) {
  const int K = c->K;
  const int64_t n = c->n;
  const size_t vb = sizeof(double) * (size_t)(n * K);
  KR_VEC(rt);
  KR_VEC(p);
  KR_VEC(pt);
  KR_VEC(q);
  KR_VEC(qt);
  double rho[4], sigma[4], alpha[4], ma[4], rn[4], rho_next[4], beta[4], t[4];
  int64_t k;
  memcpy(rt, r, vb);
  memcpy(p, r, vb);
  memcpy(pt, rt, vb);
  vdot(K, n, rt, r, rho);
  for (k = 1; k <= max_iters; ++k) {
    if (kr_tiny(orc_to_double(K, rho), c->floor)) KR_BREAK(3, k - 1);
    kr_apply(c, p, q);
    kr_apply_t(c, pt, qt);
    vdot(K, n, pt, q, sigma);
    if (kr_tiny(orc_to_double(K, sigma), c->floor)) KR_BREAK(4, k - 1);
    orc_div(K, rho, sigma, alpha);
    kr_neg(K, alpha, ma);
    kr_axpy(K, n, alpha, p, x);
    kr_axpy(K, n, ma, q, r);
    kr_axpy(K, n, ma, qt, rt);
    kr_norm2(K, n, r, rn);
    KR_RECORD(rn);
    vdot(K, n, rt, r, rho_next);
    orc_div(K, rho_next, rho, beta);
    for (int64_t i = 0; i < n; ++i) {
      orc_mul(K, beta, p + i * K, t);
      orc_add(K, r + i * K, t, p + i * K);
      orc_mul(K, beta, pt + i * K, t);
      orc_add(K, rt + i * K, t, pt + i * K);
    }
    memcpy(rho, rho_next, sizeof(rho));
  }
  *status = 1;
  *iters = max_iters;
out:
  free(rt);
  free(p);
  free(pt);
  free(q);
  free(qt);
}

static void kr_cgs(KrCtx *c, double *x, double *r, int64_t max_iters, int64_t *iters, int *status,
                   int *reason) {
  const int K = c->K;
  const int64_t n = c->n;
  const size_t vb = sizeof(double) * (size_t)(n * K);
  KR_VEC(rt);
  KR_VEC(u);
  KR_VEC(p);
  KR_VEC(q);
  KR_VEC(v);
  KR_VEC(tv);
  KR_VEC(w);
  double rho[4], sigma[4], alpha[4], ma[4], rn[4], rho_next[4], beta[4], t[4], t2[4];
  int64_t k;
  memcpy(rt, r, vb);
  memcpy(u, r, vb);
  memcpy(p, r, vb);
  vdot(K, n, rt, r, rho);
  for (k = 1; k <= max_iters; ++k) {
    if (kr_tiny(orc_to_double(K, rho), c->floor)) KR_BREAK(3, k - 1);
    kr_apply(c, p, v);
    vdot(K, n, rt, v, sigma);
    if (kr_tiny(orc_to_double(K, sigma), c->floor)) KR_BREAK(5, k - 1);
    orc_div(K, rho, sigma, alpha);
    for (int64_t i = 0; i < n; ++i) { /* q = u - alpha v; t = u + q */
      orc_mul(K, alpha, v + i * K, t);
      orc_sub(K, u + i * K, t, q + i * K);
      orc_add(K, u + i * K, q + i * K, tv + i * K);
    }
    kr_axpy(K, n, alpha, tv, x);
    kr_apply(c, tv, w);
    kr_neg(K, alpha, ma);
    kr_axpy(K, n, ma, w, r);
    kr_norm2(K, n, r, rn);
    KR_RECORD(rn);
    vdot(K, n, rt, r, rho_next);
    orc_div(K, rho_next, rho, beta);
    for (int64_t i = 0; i < n; ++i) { /* u = r + beta q; p = u + beta (q + beta p) */
      orc_mul(K, beta, q + i * K, t);
      orc_add(K, r + i * K, t, u + i * K);
      orc_mul(K, beta, p + i * K, t);
      orc_add(K, q + i * K, t, t2);
      orc_mul(K, beta, t2, t);
      orc_add(K, u + i * K, t, p + i * K);
    }
    memcpy(rho, rho_next, sizeof(rho));
  }
  *status = 1;
  *iters = max_iters;
out:
  free(rt);
  free(u);
  free(p);
  free(q);
  free(v);
  free(tv);
  free(w);
}

static void kr_bicgstab(KrCtx *c, double *x, double *r, int64_t max_iters, int64_t *iters, int *status,
                        int *reason) {
  const int K = c->K;
  const int64_t n = c->n;
  const size_t vb = sizeof(double) * (size_t)(n * K);
  KR_VEC(rt);
  KR_VEC(p);
  KR_VEC(v);
  KR_VEC(s);
  KR_VEC(tv);
  double rho[4], sigma[4], alpha[4], ma[4], rn[4], sn[4], tt[4], ts[4], omega[4], mo[4], rho_next[4],
      beta[4], q1[4], q2[4], t[4], t2[4];
  int64_t k;
  memcpy(rt, r, vb);
  memcpy(p, r, vb);
  vdot(K, n, rt, r, rho);
  for (k = 1; k <= max_iters; ++k) {
    if (kr_tiny(orc_to_double(K, rho), c->floor)) KR_BREAK(3, k - 1);
    kr_apply(c, p, v);
    vdot(K, n, rt, v, sigma);
    if (kr_tiny(orc_to_double(K, sigma), c->floor)) KR_BREAK(5, k - 1);
    orc_div(K, rho, sigma, alpha);
    kr_neg(K, alpha, ma);
    memcpy(s, r, vb);
    kr_axpy(K, n, ma, v, s);
    kr_norm2(K, n, s, sn);
    if (kr_le(K, sn, c->thr)) { /* half step converged (krylov.hpp:449-458) */
      kr_axpy(K, n, alpha, p, x);
      memcpy(r, s, vb);
      c->hist[c->nh++] = orc_to_double(K, sn);
      *status = 0;
      *reason = 0;
      *iters = k;
      goto out;
    }
    kr_apply(c, s, tv);
    vdot(K, n, tv, tv, tt);
    if (kr_tiny(orc_to_double(K, tt), c->floor)) KR_BREAK(6, k - 1);
    vdot(K, n, tv, s, ts);
    orc_div(K, ts, tt, omega);
    if (kr_tiny(orc_to_double(K, omega), c->floor)) KR_BREAK(7, k - 1);
    kr_axpy(K, n, alpha, p, x);
    kr_axpy(K, n, omega, s, x);
    memcpy(r, s, vb);
    kr_neg(K, omega, mo);
    kr_axpy(K, n, mo, tv, r);
    kr_norm2(K, n, r, rn);
    KR_RECORD(rn);
    vdot(K, n, rt, r, rho_next);
    orc_div(K, rho_next, rho, q1);
    orc_div(K, alpha, omega, q2);
    orc_mul(K, q1, q2, beta);
    for (int64_t i = 0; i < n; ++i) { /* p = r + beta (p - omega v) */
      orc_mul(K, omega, v + i * K, t);
      orc_sub(K, p + i * K, t, t2);
      orc_mul(K, beta, t2, t);
      orc_add(K, r + i * K, t, p + i * K);
    }
    memcpy(rho, rho_next, sizeof(rho));
  }
  *status = 1;
  *iters = max_iters;
out:
  free(rt);
  free(p);
  free(v);
  free(s);
  free(tv);
}

static void kr_gpbicg(KrCtx *c, double *x, double *r, int64_t max_iters, int64_t *iters, int *status,
                      int *reason) {
  const int K = c->K;
  const int64_t n = c->n;
  const size_t vb = sizeof(double) * (size_t)(n * K);
  KR_VEC(rt);
  KR_VEC(p);
  KR_VEC(tp);
  KR_VEC(w);
  KR_VEC(u);
  KR_VEC(z);
  KR_VEC(y);
  KR_VEC(ap);
  KR_VEC(tv);
  KR_VEC(at);
  double rho[4], sigma[4], alpha[4], ma[4], rn[4], tn[4], att[4], ata[4], yy[4], yat[4], yt[4], zeta[4],
      eta[4], me[4], mz[4], rho_next[4], beta[4] = {0, 0, 0, 0}, d[4], e1[4], e2[4], t[4], t2[4], t3[4];
  int64_t k;
  memcpy(rt, r, vb);
  memcpy(p, r, vb);
  vdot(K, n, rt, r, rho);
  for (k = 1; k <= max_iters; ++k) {
    if (kr_tiny(orc_to_double(K, rho), c->floor)) KR_BREAK(3, k - 1);
    kr_apply(c, p, ap);
    vdot(K, n, rt, ap, sigma);
    if (kr_tiny(orc_to_double(K, sigma), c->floor)) KR_BREAK(5, k - 1);
    orc_div(K, rho, sigma, alpha);
    for (int64_t i = 0; i < n; ++i) { /* y = (t_prev - r) + alpha (Ap - w) */
      orc_sub(K, tp + i * K, r + i * K, t);
      orc_sub(K, ap + i * K, w + i * K, t2);
      orc_mul(K, alpha, t2, t3);
      orc_add(K, t, t3, y + i * K);
    }
    kr_neg(K, alpha, ma);
    memcpy(tv, r, vb);
    kr_axpy(K, n, ma, ap, tv);
    kr_norm2(K, n, tv, tn);
    if (kr_le(K, tn, c->thr)) { /* half step converged (krylov.hpp:507-515) */
      kr_axpy(K, n, alpha, p, x);
      memcpy(r, tv, vb);
      c->hist[c->nh++] = orc_to_double(K, tn);
      *status = 0;
      *reason = 0;
      *iters = k;
      goto out;
    }
    kr_apply(c, tv, at);
    vdot(K, n, at, tv, att);
    vdot(K, n, at, at, ata);
    if (k == 1) {
      if (kr_tiny(orc_to_double(K, ata), c->floor)) KR_BREAK(8, k - 1);
      orc_div(K, att, ata, zeta);
      for (int j = 0; j < K; ++j) eta[j] = 0.0;
    } else {
      vdot(K, n, y, y, yy);
      vdot(K, n, y, at, yat);
      vdot(K, n, y, tv, yt);
      orc_mul(K, ata, yy, e1);
      orc_mul(K, yat, yat, e2);
      orc_sub(K, e1, e2, d);
      if (kr_tiny(orc_to_double(K, d), c->floor * c->floor)) KR_BREAK(9, k - 1);
      orc_mul(K, yy, att, e1);
      orc_mul(K, yt, yat, e2);
      orc_sub(K, e1, e2, t);
      orc_div(K, t, d, zeta);
      orc_mul(K, ata, yt, e1);
      orc_mul(K, yat, att, e2);
      orc_sub(K, e1, e2, t);
      orc_div(K, t, d, eta);
    }
    for (int64_t i = 0; i < n; ++i) { /* u = zeta Ap + eta ((t_prev - r) + beta u) */
      orc_sub(K, tp + i * K, r + i * K, t);
      orc_mul(K, beta, u + i * K, t2);
      orc_add(K, t, t2, t3);
      orc_mul(K, eta, t3, t);
      orc_mul(K, zeta, ap + i * K, t2);
      orc_add(K, t2, t, u + i * K);
    }
    for (int64_t i = 0; i < n; ++i) { /* z = (zeta r + eta z) - alpha u */
      orc_mul(K, zeta, r + i * K, t);
      orc_mul(K, eta, z + i * K, t2);
      orc_add(K, t, t2, t3);
      orc_mul(K, alpha, u + i * K, t);
      orc_sub(K, t3, t, z + i * K);
    }
    kr_axpy(K, n, alpha, p, x);
    for (int64_t i = 0; i < n; ++i) orc_add(K, x + i * K, z + i * K, x + i * K);
    memcpy(r, tv, vb); /* r = t - eta y - zeta At */
    kr_neg(K, eta, me);
    kr_neg(K, zeta, mz);
    kr_axpy(K, n, me, y, r);
    kr_axpy(K, n, mz, at, r);
    kr_norm2(K, n, r, rn);
    KR_RECORD(rn);
    vdot(K, n, rt, r, rho_next);
    if (kr_tiny(orc_to_double(K, zeta), c->floor)) KR_BREAK(10, k);
    orc_div(K, alpha, zeta, e1);
    orc_div(K, rho_next, rho, e2);
    orc_mul(K, e1, e2, beta);
    for (int64_t i = 0; i < n; ++i) { /* w = At + beta Ap; p = r + beta (p - u) */
      orc_mul(K, beta, ap + i * K, t);
      orc_add(K, at + i * K, t, w + i * K);
      orc_sub(K, p + i * K, u + i * K, t);
      orc_mul(K, beta, t, t2);
      orc_add(K, r + i * K, t2, p + i * K);
    }
    memcpy(tp, tv, vb);
    memcpy(rho, rho_next, sizeof(rho));
  }
  *status = 1;
  *iters = max_iters;
out:
  free(rt);
  free(p);
  free(tp);
  free(w);
  free(u);
  free(z);
  free(y);
  free(ap);
  free(tv);
  free(at);
}

/* solve() (krylov.hpp:596-606).  x0 may be NULL (zero start).  history needs
 * max_iters + 1 entries.  Returns the history length, or -1 on a config error
 * (SolverConfig::validate, krylov.hpp:69-75). */
ORC_API int orc_solve_ex(int method, int K, int lanes, int threads, int mixed, int64_t n, const int64_t *indptr,
                         const int64_t *indices, const double *vals, const double *b, const double *x0,
                         double rel_tol, double abs_tol, int64_t max_iters, double *x, double *history,
                         int64_t *iterations, int *status, int *reason, double *rhs_norm,
                         double *final_true_residual);

ORC_API int orc_solve(int method, int K, int lanes, int threads, int64_t n, const int64_t *indptr,
                      const int64_t *indices, const double *vals, const double *b, const double *x0,
                      double rel_tol, double abs_tol, int64_t max_iters, double *x, double *history,
                      int64_t *iterations, int *status, int *reason, double *rhs_norm,
                      double *final_true_residual) {
  return orc_solve_ex(method, K, lanes, threads, 0, n, indptr, indices, vals, b, x0, rel_tol, abs_tol, max_iters,
                      x, history, iterations, status, reason, rhs_norm, final_true_residual);
}

/* mixed != 0: vals is the binary64 matrix (one plane), products mul_by_double
 * (Mixed mode, kernels.hpp:55-58) -- solve() over CsrOperator<double>. */
ORC_API int orc_solve_ex(int method, int K, int lanes, int threads, int mixed, int64_t n, const int64_t *indptr,
                         const int64_t *indices, const double *vals, const double *b, const double *x0,
                         double rel_tol, double abs_tol, int64_t max_iters, double *x, double *history,
                         int64_t *iterations, int *status, int *reason, double *rhs_norm,
                         double *final_true_residual) {
  if (!(rel_tol > 0.0) || !(abs_tol > 0.0) || max_iters < 1 || method < 0 || method > 4) return -1;
  KrCtx c = {K, lanes, threads < 1 ? 1 : threads, n, indptr, indices, vals, {0, 0, 0, 0}, 0, 0, history, 0,
             mixed ? 1 : 0};
  KR_VEC(r);
  KR_VEC(q);
  double t[4], bn[4], tmp[4], r0[4];
  for (int64_t i = 0; i < n * K; ++i) x[i] = 0.0;
  if (x0) { /* x = scalar_like(x0); r = b - A x (krylov.hpp:174-181) */
    for (int64_t i = 0; i < n; ++i) x[i * K] = x0[i];
    kr_apply(&c, x, q);
    for (int64_t i = 0; i < n; ++i) orc_sub(K, b + i * K, q + i * K, r + i * K);
  } else {
    memcpy(r, b, sizeof(double) * (size_t)(n * K));
  }
  kr_norm2(K, n, b, bn);
  orc_mul_d(K, bn, rel_tol, tmp);
  double at[4] = {abs_tol, 0, 0, 0};
  orc_add(K, tmp, at, c.thr);
  *rhs_norm = orc_to_double(K, bn);
  c.cap = 1e6 * *rhs_norm + 1e6 * abs_tol;
  c.floor = 1e-3 * abs_tol;
  kr_norm2(K, n, r, r0);
  history[c.nh++] = orc_to_double(K, r0);
  *reason = 0;
  if (kr_le(K, r0, c.thr)) {
    *status = 0;
    *iterations = 0;
  } else {
    void (*fn[5])(KrCtx *, double *, double *, int64_t, int64_t *, int *, int *) = {
        kr_cg, kr_bicg, kr_cgs, kr_bicgstab, kr_gpbicg};
    fn[method](&c, x, r, max_iters, iterations, status, reason);
  }
  kr_apply(&c, x, q); /* finish_true_residual */
  for (int64_t i = 0; i < n; ++i) orc_sub(K, b + i * K, q + i * K, q + i * K);
  kr_norm2(K, n, q, t);
  *final_true_residual = orc_to_double(K, t);
  free(r);
  free(q);
  return (int)c.nh;
}
