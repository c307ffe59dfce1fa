// mc_arith.cuh -- sm_100a device multi-component (DD/TD/QD) arithmetic.
//
// Op-for-op restatement of the reference arithmetic so the deterministic
// kernels reproduce its bits (paths under /root/reference/proj/include/mps/):
//   eft.hpp:26-80        quick_two_sum_raw, two_sum, two_prod_fma, three_sum(2)
//   multicomp.hpp:43-78  renorm_n<K,N> (branchy forward collect kept exactly)
//   multicomp.hpp:80-215 DD cores, QD sloppy prenorms, TD-as-zero-extended-QD
//   multicomp.hpp:225-335 add / mul / mul_by_double / sub / divide / sqrt /
//                         to_double / compare
// Every arithmetic step is an explicit round-to-nearest intrinsic
// (__dadd_rn, __dsub_rn, __dmul_rn, __fma_rn), so no compiler flag can contract
// or reassociate them; fma appears only where the reference calls std::fma
// (eft.hpp:57, multicomp.hpp:106).  Values live in registers as MC<K>
// (K doubles, magnitude-decreasing).
#pragma once

#include <cstdint>

namespace mpsg {

template <int K>
struct MC {
  double c[K];
};

#define MPSG_DI __device__ __forceinline__

MPSG_DI double dadd(double a, double b) { return __dadd_rn(a, b); }
MPSG_DI double dsub(double a, double b) { return __dsub_rn(a, b); }
MPSG_DI double dmul(double a, double b) { return __dmul_rn(a, b); }
MPSG_DI double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// Bit tests on the integer pipe instead of DSETP on the fp64 pipe.
// x != 0.0 (false for +-0, true for NaN), multicomp.hpp:68.
MPSG_DI bool nonzero(double x) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b << 1) != 0ull;
}
// std::isfinite, multicomp.hpp:47.
MPSG_DI bool finite(double x) {
  return (__double2hiint(x) & 0x7ff00000) != 0x7ff00000;
}

// ---------------------------------------------------------------- EFTs --
MPSG_DI void qts(double a, double b, double& s, double& e) {  // eft.hpp:26-30
  double ss = dadd(a, b);
  e = dsub(b, dsub(ss, a));
  s = ss;
}
MPSG_DI void two_sum(double a, double b, double& s, double& e) {  // eft.hpp:34-41
  double ss = dadd(a, b);
  double v = dsub(ss, a);
  e = dadd(dsub(a, dsub(ss, v)), dsub(b, v));
  s = ss;
}
MPSG_DI void two_prod(double a, double b, double& p, double& e) {  // eft.hpp:53-59
  double pp = dmul(a, b);
  e = dfma(a, b, -pp);
  p = pp;
}
MPSG_DI void three_sum(double& a, double& b, double& c) {  // eft.hpp:63-71
  double t1, t2, s1, t3, s2, s3;
  two_sum(a, b, t1, t2);
  two_sum(c, t1, s1, t3);
  two_sum(t2, t3, s2, s3);
  a = s1;
  b = s2;
  c = s3;
}
MPSG_DI void three_sum2(double& a, double& b, double c) {  // eft.hpp:74-80
  double t1, t2, s1, t3;
  two_sum(a, b, t1, t2);
  two_sum(c, t1, s1, t3);
  a = s1;
  b = dadd(t2, t3);
}

// ------------------------------------------------------------ renorm_n --
// multicomp.hpp:43-78.  t[] is taken by value in registers.
//
// The forward collect emits a component whenever QuickTwoSum leaves a
// nonzero low part.  On full-precision data every one of the first K-1 steps
// emits (the "common path": K-1 QuickTwoSums, then plain adds), so that path
// is computed straight-line and only if one of its low parts is zero does the
// general collect below run -- a warp-uniform branch on uniform data that
// yields exactly the values of the reference's loop either way.
// Zero tests use integer ops on the bit pattern (x != 0.0, true for NaN).
MPSG_DI bool nonzero_i(double x) {
  return ((__double2hiint(x) & 0x7fffffff) | __double2loint(x)) != 0;
}

template <int K, int N>
MPSG_DI void renorm_general(double (&t)[N], MC<K>& r) {
#pragma unroll
  for (int i = 0; i < K; ++i) r.c[i] = 0.0;
  int k = 0;
  double s = t[0];
#pragma unroll
  for (int i = 1; i < N; ++i) {
    if (k == K - 1) {
      s = dadd(s, t[i]);
    } else {
      double hi, lo;
      qts(s, t[i], hi, lo);
      if (nonzero_i(lo)) {
#pragma unroll
        for (int j = 0; j < K - 1; ++j)
          if (k == j) r.c[j] = hi;
        ++k;
        s = lo;
      } else {
        s = hi;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (k == j) r.c[j] = s;
}

template <int K, int N>
MPSG_DI MC<K> renorm(double (&t)[N]) {
  MC<K> r;
  if (!finite(t[0])) {
#pragma unroll
    for (int i = 0; i < K; ++i) r.c[i] = 0.0;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s = dadd(s, t[i]);
    r.c[0] = s;
    return r;
  }
  double s = t[N - 1];
#pragma unroll
  for (int i = N - 2; i >= 0; --i) {
    double hi, lo;
    qts(t[i], s, hi, lo);
    s = hi;
    t[i + 1] = lo;
  }
  t[0] = s;
  // common path
  bool ok = true;
#pragma unroll
  for (int i = 1; i < K; ++i) {
    double hi, lo;
    qts(s, t[i], hi, lo);
    r.c[i - 1] = hi;
    s = lo;
    ok = ok && nonzero_i(lo);
  }
#pragma unroll
  for (int i = K; i < N; ++i) s = dadd(s, t[i]);
  r.c[K - 1] = s;
  if (__builtin_expect(ok, 1)) return r;
  renorm_general<K, N>(t, r);
  return r;
}

// ------------------------------------------------------------ DD cores --
MPSG_DI MC<2> dd_add(const MC<2>& x, const MC<2>& y) {  // multicomp.hpp:80-88
  double s, e;
  two_sum(x.c[0], y.c[0], s, e);
  double w = dadd(x.c[1], y.c[1]);
  e = dadd(e, w);
  MC<2> r;
  qts(s, e, r.c[0], r.c[1]);
  return r;
}
MPSG_DI MC<2> dd_mul(const MC<2>& x, const MC<2>& y) {  // multicomp.hpp:90-100
  double p1, p2;
  two_prod(x.c[0], y.c[0], p1, p2);
  double w1 = dmul(x.c[0], y.c[1]);
  double w2 = dmul(x.c[1], y.c[0]);
  double w3 = dadd(w1, w2);
  p2 = dadd(p2, w3);
  MC<2> r;
  qts(p1, p2, r.c[0], r.c[1]);
  return r;
}
MPSG_DI MC<2> dd_mul_d(const MC<2>& x, double y) {  // multicomp.hpp:102-110
  double p1, p2;
  two_prod(x.c[0], y, p1, p2);
  p2 = dfma(x.c[1], y, p2);
  MC<2> r;
  qts(p1, p2, r.c[0], r.c[1]);
  return r;
}

// ----------------------------------------------------- QD/TD prenorms --
// multicomp.hpp:112-132
MPSG_DI void qd_add_prenorm(const double* x, const double* y, double* out) {
  double s0, t0, s1, t1, s2, t2, s3, t3;
  two_sum(x[0], y[0], s0, t0);
  two_sum(x[1], y[1], s1, t1);
  two_sum(x[2], y[2], s2, t2);
  two_sum(x[3], y[3], s3, t3);
  double s1b, t0b;
  two_sum(s1, t0, s1b, t0b);
  s1 = s1b;
  t0 = t0b;
  three_sum(s2, t0, t1);
  three_sum2(s3, t0, t2);
  t0 = dadd(dadd(t0, t1), t3);
  out[0] = s0;
  out[1] = s1;
  out[2] = s2;
  out[3] = s3;
  out[4] = t0;
}
// multicomp.hpp:134-163
MPSG_DI void qd_mul_prenorm(const double* a, const double* b, double* out) {
  double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5;
  two_prod(a[0], b[0], p0, q0);
  two_prod(a[0], b[1], p1, q1);
  two_prod(a[1], b[0], p2, q2);
  two_prod(a[0], b[2], p3, q3);
  two_prod(a[1], b[1], p4, q4);
  two_prod(a[2], b[0], p5, q5);
  three_sum(p1, p2, q0);
  three_sum(p2, q1, q2);
  three_sum(p3, p4, p5);
  double s0, t0, s1, t1;
  two_sum(p2, p3, s0, t0);
  two_sum(q1, p4, s1, t1);
  double s2 = dadd(q2, p5);
  double s1b, t0b;
  two_sum(s1, t0, s1b, t0b);
  s1 = s1b;
  s2 = dadd(s2, dadd(t0b, t1));
  // multicomp.hpp:156, strictly left to right with separate multiplies
  double tail = dadd(dmul(a[0], b[3]), dmul(a[1], b[2]));
  tail = dadd(tail, dmul(a[2], b[1]));
  tail = dadd(tail, dmul(a[3], b[0]));
  tail = dadd(tail, q0);
  tail = dadd(tail, q3);
  tail = dadd(tail, q4);
  tail = dadd(tail, q5);
  s1 = dadd(s1, tail);
  out[0] = p0;
  out[1] = p1;
  out[2] = s0;
  out[3] = s1;
  out[4] = s2;
}
// multicomp.hpp:165-183
MPSG_DI void qd_mul_d_prenorm(const double* a, double b, double* out) {
  double p0, q0, p1, q1, p2, q2;
  two_prod(a[0], b, p0, q0);
  two_prod(a[1], b, p1, q1);
  two_prod(a[2], b, p2, q2);
  double p3 = dmul(a[3], b);
  double s1, s2;
  two_sum(q0, p1, s1, s2);
  three_sum(s2, q1, p2);
  three_sum2(q1, p2, p3);
  out[0] = p0;
  out[1] = s1;
  out[2] = s2;
  out[3] = q1;
  out[4] = dadd(q2, p2);
}
// multicomp.hpp:185-199
MPSG_DI void td_mul_d_prenorm(const double* a, double b, double* out) {
  double p0, q0, p1, q1, p2, q2;
  two_prod(a[0], b, p0, q0);
  two_prod(a[1], b, p1, q1);
  two_prod(a[2], b, p2, q2);
  double s1, s2;
  two_sum(q0, p1, s1, s2);
  three_sum(s2, q1, p2);
  out[0] = p0;
  out[1] = s1;
  out[2] = s2;
  out[3] = dadd(q2, p2);
}

// ------------------------------------------------ public MC operations --
// multicomp.hpp:225-277 (add / mul / mul_by_double per width)
MPSG_DI MC<2> add(const MC<2>& x, const MC<2>& y) { return dd_add(x, y); }
MPSG_DI MC<2> mul(const MC<2>& x, const MC<2>& y) { return dd_mul(x, y); }
MPSG_DI MC<2> mul_d(const MC<2>& x, double y) { return dd_mul_d(x, y); }

MPSG_DI MC<3> add(const MC<3>& x, const MC<3>& y) {  // multicomp.hpp:243-247, :203-207
  double xe[4] = {x.c[0], x.c[1], x.c[2], 0.0};
  double ye[4] = {y.c[0], y.c[1], y.c[2], 0.0};
  double t[5];
  qd_add_prenorm(xe, ye, t);
  return renorm<3, 5>(t);
}
MPSG_DI MC<3> mul(const MC<3>& x, const MC<3>& y) {  // multicomp.hpp:249-253, :210-214
  double xe[4] = {x.c[0], x.c[1], x.c[2], 0.0};
  double ye[4] = {y.c[0], y.c[1], y.c[2], 0.0};
  double t[5];
  qd_mul_prenorm(xe, ye, t);
  return renorm<3, 5>(t);
}
MPSG_DI MC<3> mul_d(const MC<3>& x, double y) {  // multicomp.hpp:255-259
  double t[4];
  td_mul_d_prenorm(x.c, y, t);
  return renorm<3, 4>(t);
}
MPSG_DI MC<4> add(const MC<4>& x, const MC<4>& y) {  // multicomp.hpp:261-265
  double t[5];
  qd_add_prenorm(x.c, y.c, t);
  return renorm<4, 5>(t);
}
MPSG_DI MC<4> mul(const MC<4>& x, const MC<4>& y) {  // multicomp.hpp:267-271
  double t[5];
  qd_mul_prenorm(x.c, y.c, t);
  return renorm<4, 5>(t);
}
MPSG_DI MC<4> mul_d(const MC<4>& x, double y) {  // multicomp.hpp:273-277
  double t[5];
  qd_mul_d_prenorm(x.c, y, t);
  return renorm<4, 5>(t);
}

// ---------------------------------------------------------------------------
// FAST-mode product-accumulate acc + a*x (SURVEY 8(a) hard part 2: "the fast
// mode may fuse mul+add into one renormalisation per nnz, provided the
// componentwise bound holds").  Not the reference's bits; every use is checked
// against |y - y_ref| <= 4 rowlen u sum|a||x| (tests/test_gpu_spmv.py,
// tools/fused_probe.py, tools/fused_adversarial.py).
//  * fma_fast: the product's five pre-normalisation terms (qd_mul_prenorm, the
//    last two merged) straight into qd_add_prenorm, then the add's full
//    renorm_n -- skips the product's own renormalisation.  Used where the
//    result is stored (vector updates).
//  * fma_acc: the running row / dot accumulator, summed level by level
//    (MPSG_QD_LEVELS, below) and kept by a backward quick-two-sum sweep only
//    (the forward collect that canonicalises zero components is left to
//    canon() once per row): QD 121 and TD 52 fp64 operations per nonzero
//    instead of 206 / 202; worst 0.15 (QD) / 0.18 (TD) of the bound on the
//    adversarial probes (long rows, 2^+-60 exponent spread, exact
//    cancellation).  MPSG_QD_LEVELS=0 builds the previous prenorm-chained
//    accumulate (QD 176 operations, worst 0.009).
// ---------------------------------------------------------------------------
MPSG_DI MC<4> renorm_sweep(double (&t)[5]) {  // renorm_n<4,5>'s backward sweep, tail merged
  double s = t[4];
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    double hi, lo;
    qts(t[i], s, hi, lo);
    s = hi;
    t[i + 1] = lo;
  }
  MC<4> r;
  r.c[0] = s;
  r.c[1] = t[1];
  r.c[2] = t[2];
  r.c[3] = dadd(t[3], t[4]);
  return r;
}
template <bool SWEEP>
MPSG_DI MC<4> qd_fused(const MC<4>& acc, const double (&pv)[4]) {
  double t[5];
  qd_add_prenorm(acc.c, pv, t);
  if constexpr (SWEEP)
    return renorm_sweep(t);
  else
    return renorm<4, 5>(t);
}
#ifndef MPSG_QD_LEVELS
#define MPSG_QD_LEVELS 1
#endif
MPSG_DI MC<4> canon(const MC<4>& v);
MPSG_DI MC<3> canon(const MC<3>& v);
#if MPSG_QD_LEVELS
MPSG_DI MC<4> fma_acc(const MC<4>& acc, const MC<4>& a, const MC<4>& x);
MPSG_DI MC<3> fma_acc(const MC<3>& acc, const MC<3>& a, const MC<3>& x);
// stored updates: the level-wise accumulate, then the full renormalisation
// (QD 121 + 22, TD 52 + 16 operations instead of 185 / 183)
MPSG_DI MC<4> fma_fast(const MC<4>& acc, const MC<4>& a, const MC<4>& x) { return canon(fma_acc(acc, a, x)); }
#else
MPSG_DI MC<4> fma_fast(const MC<4>& acc, const MC<4>& a, const MC<4>& x) {
  double p[5];
  qd_mul_prenorm(a.c, x.c, p);
  const double pv[4] = {p[0], p[1], p[2], dadd(p[3], p[4])};
  return qd_fused<false>(acc, pv);
}
#endif
#if MPSG_QD_LEVELS
// Level-wise QD product-accumulate: acc + a*x summed by magnitude level
// (level k = terms of order 2^-53k): each level's terms chained through
// two_sums whose errors drop to the next level; level 3 is a plain sum, small
// terms first and the accumulator's own c3 last; then the backward sweep.
// 121 fp64 operations instead of 176 (product and add prenorms + sweep).
// The dropped terms are the ones the reference's qd_mul_prenorm drops
// (a1x3, a2x2, a3x1 and the errors of the order-3 products).
MPSG_DI MC<4> fma_acc(const MC<4>& acc, const MC<4>& a, const MC<4>& x) {
  double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5;
  two_prod(a.c[0], x.c[0], p0, q0);
  two_prod(a.c[0], x.c[1], p1, q1);
  two_prod(a.c[1], x.c[0], p2, q2);
  two_prod(a.c[0], x.c[2], p3, q3);
  two_prod(a.c[1], x.c[1], p4, q4);
  two_prod(a.c[2], x.c[0], p5, q5);
  double s0, e0, u, f1, f2, f3, f4, s1, v, g[9], s2;
  two_sum(acc.c[0], p0, s0, e0);  // level 0
  two_sum(acc.c[1], p1, u, f1);   // level 1: c1 p1 p2 q0 e0
  two_sum(u, p2, u, f2);
  two_sum(u, q0, u, f3);
  two_sum(u, e0, s1, f4);
  two_sum(acc.c[2], p3, v, g[0]);  // level 2: c2 p3 p4 p5 q1 q2 f1..f4
  two_sum(v, p4, v, g[1]);
  two_sum(v, p5, v, g[2]);
  two_sum(v, q1, v, g[3]);
  two_sum(v, q2, v, g[4]);
  two_sum(v, f1, v, g[5]);
  two_sum(v, f2, v, g[6]);
  two_sum(v, f3, v, g[7]);
  two_sum(v, f4, s2, g[8]);
  double w = g[0];  // level 3
#pragma unroll
  for (int i = 1; i < 9; ++i) w = dadd(w, g[i]);
  w = dadd(dadd(dadd(w, q3), q4), q5);
  w = dfma(a.c[0], x.c[3], w);
  w = dfma(a.c[1], x.c[2], w);
  w = dfma(a.c[2], x.c[1], w);
  w = dfma(a.c[3], x.c[0], w);
  w = dadd(w, acc.c[3]);
  MC<4> r;
  double h;
  qts(s2, w, h, r.c[3]);
  qts(s1, h, h, r.c[2]);
  qts(s0, h, r.c[0], r.c[1]);
  return r;
}
#else
MPSG_DI MC<4> fma_acc(const MC<4>& acc, const MC<4>& a, const MC<4>& x) {
  double p[5];
  qd_mul_prenorm(a.c, x.c, p);
  const double pv[4] = {p[0], p[1], p[2], dadd(p[3], p[4])};
  return qd_fused<true>(acc, pv);
}
#endif
#if MPSG_QD_LEVELS
MPSG_DI MC<3> fma_fast(const MC<3>& acc, const MC<3>& a, const MC<3>& x) { return canon(fma_acc(acc, a, x)); }
#else
MPSG_DI MC<3> fma_fast(const MC<3>& acc, const MC<3>& a, const MC<3>& x) {
  const double ae[4] = {a.c[0], a.c[1], a.c[2], 0.0};
  const double xe[4] = {x.c[0], x.c[1], x.c[2], 0.0};
  double p[5];
  qd_mul_prenorm(ae, xe, p);
  const double pv[4] = {p[0], p[1], p[2], dadd(p[3], p[4])};
  const double ce[4] = {acc.c[0], acc.c[1], acc.c[2], 0.0};
  double t[5];
  qd_add_prenorm(ce, pv, t);
  return renorm<3, 5>(t);
}
#endif
#ifndef MPSG_TD_SWEEP
#define MPSG_TD_SWEEP 1
#endif
#if MPSG_QD_LEVELS
// Level-wise TD product-accumulate (as the QD one above, one level fewer):
// levels 0-1 through two_sums, level 2 a plain sum (small terms first, the
// accumulator's c2 last), then the backward sweep.  52 fp64 operations instead
// of 177 (the reference's TD runs the QD chains on zero-extended operands).
MPSG_DI MC<3> fma_acc(const MC<3>& acc, const MC<3>& a, const MC<3>& x) {
  double p0, q0, p1, q1, p2, q2;
  two_prod(a.c[0], x.c[0], p0, q0);
  two_prod(a.c[0], x.c[1], p1, q1);
  two_prod(a.c[1], x.c[0], p2, q2);
  double s0, e0, u, f1, f2, f3, f4, s1;
  two_sum(acc.c[0], p0, s0, e0);  // level 0
  two_sum(acc.c[1], p1, u, f1);   // level 1: c1 p1 p2 q0 e0
  two_sum(u, p2, u, f2);
  two_sum(u, q0, u, f3);
  two_sum(u, e0, s1, f4);
  double w = dadd(dadd(dadd(dadd(dadd(f1, f2), f3), f4), q1), q2);  // level 2
  w = dfma(a.c[0], x.c[2], w);
  w = dfma(a.c[1], x.c[1], w);
  w = dfma(a.c[2], x.c[0], w);
  w = dadd(w, acc.c[2]);
  MC<3> r;
  double h;
  qts(s1, w, h, r.c[2]);
  qts(s0, h, r.c[0], r.c[1]);
  return r;
}
#else
MPSG_DI MC<3> fma_acc(const MC<3>& acc, const MC<3>& a, const MC<3>& x) {
#if MPSG_TD_SWEEP
  const double ae[4] = {a.c[0], a.c[1], a.c[2], 0.0};
  const double xe[4] = {x.c[0], x.c[1], x.c[2], 0.0};
  double p[5];
  qd_mul_prenorm(ae, xe, p);
  const double pv[4] = {p[0], p[1], p[2], dadd(p[3], p[4])};
  const double ce[4] = {acc.c[0], acc.c[1], acc.c[2], 0.0};
  double t[5];
  qd_add_prenorm(ce, pv, t);
  double s = t[4];
#pragma unroll
  for (int i = 3; i >= 0; --i) {
    double hi, lo;
    qts(t[i], s, hi, lo);
    s = hi;
    t[i + 1] = lo;
  }
  MC<3> r;
  r.c[0] = s;
  r.c[1] = t[1];
  r.c[2] = dadd(dadd(t[2], t[3]), t[4]);
  return r;
#else
  return fma_fast(acc, a, x);
#endif
}
#endif
// Level accumulators (warp-specialised short-row kernel, spmv_ws.cuh): the
// level sums (s0, u, v, w) of fma_acc kept UNNORMALISED across a short group
// of products -- every two_sum error still drops one level, so the value is
// the same exact sum up to the level-3 (level-2 for TD) roundings -- and swept
// once per group (lvl_sweep: fma_acc's three backward quick-two-sums) instead
// of once per product: QD 112 + 9/G, TD 45 + 6/G operations per nonzero
// instead of 121 / 52, and the four level chains of consecutive products are
// independent of each other (no serial dependence through the sweep).  The
// group is kept short (G = 4) so a level sum never outgrows the level above
// it by more than the few terms of one group.
MPSG_DI void fma_lvl(MC<4>& r, const MC<4>& a, const MC<4>& x) {
  double p, q, q0, q1, q2, e0, f1, f2, f3, f4, g;
  double w = r.c[3];
  two_prod(a.c[0], x.c[0], p, q0);  // level 0
  two_sum(r.c[0], p, r.c[0], e0);
  two_prod(a.c[0], x.c[1], p, q1);  // level 1: p1 p2 q0 e0
  two_sum(r.c[1], p, r.c[1], f1);
  two_prod(a.c[1], x.c[0], p, q2);
  two_sum(r.c[1], p, r.c[1], f2);
  two_sum(r.c[1], q0, r.c[1], f3);
  two_sum(r.c[1], e0, r.c[1], f4);
  two_prod(a.c[0], x.c[2], p, q);  // level 2: p3 p4 p5 q1 q2 f1..f4; errors and low parts to level 3
  two_sum(r.c[2], p, r.c[2], g);
  w = dadd(dadd(w, g), q);
  two_prod(a.c[1], x.c[1], p, q);
  two_sum(r.c[2], p, r.c[2], g);
  w = dadd(dadd(w, g), q);
  two_prod(a.c[2], x.c[0], p, q);
  two_sum(r.c[2], p, r.c[2], g);
  w = dadd(dadd(w, g), q);
  two_sum(r.c[2], q1, r.c[2], g);
  w = dadd(w, g);
  two_sum(r.c[2], q2, r.c[2], g);
  w = dadd(w, g);
  two_sum(r.c[2], f1, r.c[2], g);
  w = dadd(w, g);
  two_sum(r.c[2], f2, r.c[2], g);
  w = dadd(w, g);
  two_sum(r.c[2], f3, r.c[2], g);
  w = dadd(w, g);
  two_sum(r.c[2], f4, r.c[2], g);
  w = dadd(w, g);
  w = dfma(a.c[0], x.c[3], w);  // level 3
  w = dfma(a.c[1], x.c[2], w);
  w = dfma(a.c[2], x.c[1], w);
  w = dfma(a.c[3], x.c[0], w);
  r.c[3] = w;
}
MPSG_DI MC<4> lvl_sweep(const MC<4>& v) {
  MC<4> r;
  double h;
  qts(v.c[2], v.c[3], h, r.c[3]);
  qts(v.c[1], h, h, r.c[2]);
  qts(v.c[0], h, r.c[0], r.c[1]);
  return r;
}
MPSG_DI void fma_lvl(MC<3>& r, const MC<3>& a, const MC<3>& x) {
  double p, q0, q1, q2, e0, f1, f2, f3, f4;
  two_prod(a.c[0], x.c[0], p, q0);  // level 0
  two_sum(r.c[0], p, r.c[0], e0);
  two_prod(a.c[0], x.c[1], p, q1);  // level 1
  two_sum(r.c[1], p, r.c[1], f1);
  two_prod(a.c[1], x.c[0], p, q2);
  two_sum(r.c[1], p, r.c[1], f2);
  two_sum(r.c[1], q0, r.c[1], f3);
  two_sum(r.c[1], e0, r.c[1], f4);
  double w = dadd(dadd(dadd(dadd(dadd(dadd(r.c[2], f1), f2), f3), f4), q1), q2);  // level 2
  w = dfma(a.c[0], x.c[2], w);
  w = dfma(a.c[1], x.c[1], w);
  w = dfma(a.c[2], x.c[0], w);
  r.c[2] = w;
}
// Mixed mode (binary64 matrix value a): products x_i * a at level i.
// QD 67 + 9/G, TD 33 + 6/G operations per nonzero.
MPSG_DI void fma_lvl_d(MC<4>& r, const MC<4>& x, double a) {
  double p, q0, q1, q2, e0, f1, f2, f3, g;
  double w = r.c[3];
  two_prod(x.c[0], a, p, q0);  // level 0
  two_sum(r.c[0], p, r.c[0], e0);
  two_prod(x.c[1], a, p, q1);  // level 1: p1 q0 e0
  two_sum(r.c[1], p, r.c[1], f1);
  two_sum(r.c[1], q0, r.c[1], f2);
  two_sum(r.c[1], e0, r.c[1], f3);
  two_prod(x.c[2], a, p, q2);  // level 2: p2 q1 f1..f3
  two_sum(r.c[2], p, r.c[2], g);
  w = dadd(dadd(w, g), q2);
  two_sum(r.c[2], q1, r.c[2], g);
  w = dadd(w, g);
  two_sum(r.c[2], f1, r.c[2], g);
  w = dadd(w, g);
  two_sum(r.c[2], f2, r.c[2], g);
  w = dadd(w, g);
  two_sum(r.c[2], f3, r.c[2], g);
  w = dadd(w, g);
  r.c[3] = dfma(x.c[3], a, w);  // level 3
}
MPSG_DI void fma_lvl_d(MC<3>& r, const MC<3>& x, double a) {
  double p, q0, q1, e0, f1, f2, f3;
  two_prod(x.c[0], a, p, q0);  // level 0
  two_sum(r.c[0], p, r.c[0], e0);
  two_prod(x.c[1], a, p, q1);  // level 1
  two_sum(r.c[1], p, r.c[1], f1);
  two_sum(r.c[1], q0, r.c[1], f2);
  two_sum(r.c[1], e0, r.c[1], f3);
  const double w = dadd(dadd(dadd(dadd(r.c[2], f1), f2), f3), q1);  // level 2
  r.c[2] = dfma(x.c[2], a, w);
}
MPSG_DI MC<2> lvl_sweep(const MC<2>& v) { return v; }
// r += x on level sums (both operands may be unnormalised level sums): the
// tree combines of the FAST-order reductions -- QD 40, TD 22 operations
// instead of the full add's 85 / 83, swept and canonicalised once at the end.
MPSG_DI void lvl_add(MC<4>& r, const MC<4>& x) {
  double e0, f1, f2, g1, g2, g3;
  two_sum(r.c[0], x.c[0], r.c[0], e0);
  two_sum(r.c[1], x.c[1], r.c[1], f1);
  two_sum(r.c[1], e0, r.c[1], f2);
  two_sum(r.c[2], x.c[2], r.c[2], g1);
  two_sum(r.c[2], f1, r.c[2], g2);
  two_sum(r.c[2], f2, r.c[2], g3);
  r.c[3] = dadd(dadd(dadd(dadd(r.c[3], x.c[3]), g1), g2), g3);
}
MPSG_DI void lvl_add(MC<3>& r, const MC<3>& x) {
  double e0, f1, f2;
  two_sum(r.c[0], x.c[0], r.c[0], e0);
  two_sum(r.c[1], x.c[1], r.c[1], f1);
  two_sum(r.c[1], e0, r.c[1], f2);
  r.c[2] = dadd(dadd(dadd(r.c[2], x.c[2]), f1), f2);
}
MPSG_DI void lvl_add(MC<2>& r, const MC<2>& x) { r = add(r, x); }
MPSG_DI MC<3> lvl_sweep(const MC<3>& v) {
  MC<3> r;
  double h;
  qts(v.c[1], v.c[2], h, r.c[2]);
  qts(v.c[0], h, r.c[0], r.c[1]);
  return r;
}
// DD: the product's (p1, p2) without its quick_two_sum, straight into the add
MPSG_DI MC<2> fma_fast(const MC<2>& acc, const MC<2>& a, const MC<2>& x) {
  double p1, p2;
  two_prod(a.c[0], x.c[0], p1, p2);
  p2 = dadd(p2, dadd(dmul(a.c[0], x.c[1]), dmul(a.c[1], x.c[0])));
  double s, e;
  two_sum(acc.c[0], p1, s, e);
  e = dadd(e, dadd(acc.c[1], p2));
  MC<2> r;
  qts(s, e, r.c[0], r.c[1]);
  return r;
}
MPSG_DI MC<2> fma_acc(const MC<2>& acc, const MC<2>& a, const MC<2>& x) { return fma_fast(acc, a, x); }
// Mixed mode: acc + x*a with a binary64 matrix value (mul_by_double's
// pre-normalisation terms straight into the add)
#if MPSG_QD_LEVELS
// Mixed mode, level-wise (as fma_acc): products x_i*a at level i, 76 fp64
// operations instead of 122.
MPSG_DI MC<4> fma_acc_d(const MC<4>& acc, const MC<4>& x, double a) {
  double p0, q0, p1, q1, p2, q2;
  two_prod(x.c[0], a, p0, q0);
  two_prod(x.c[1], a, p1, q1);
  two_prod(x.c[2], a, p2, q2);
  double s0, e0, u, f1, f2, f3, s1, v, g0, g1, g2, g3, g4, s2;
  two_sum(acc.c[0], p0, s0, e0);  // level 0
  two_sum(acc.c[1], p1, u, f1);   // level 1: c1 p1 q0 e0
  two_sum(u, q0, u, f2);
  two_sum(u, e0, s1, f3);
  two_sum(acc.c[2], p2, v, g0);  // level 2: c2 p2 q1 f1..f3
  two_sum(v, q1, v, g1);
  two_sum(v, f1, v, g2);
  two_sum(v, f2, v, g3);
  two_sum(v, f3, s2, g4);
  double w = dadd(dadd(dadd(dadd(dadd(g0, g1), g2), g3), g4), q2);  // level 3
  w = dfma(x.c[3], a, w);
  w = dadd(w, acc.c[3]);
  MC<4> r;
  double h;
  qts(s2, w, h, r.c[3]);
  qts(s1, h, h, r.c[2]);
  qts(s0, h, r.c[0], r.c[1]);
  return r;
}
#else
MPSG_DI MC<4> fma_acc_d(const MC<4>& acc, const MC<4>& x, double a) {
  double p[5];
  qd_mul_d_prenorm(x.c, a, p);
  const double pv[4] = {p[0], p[1], p[2], dadd(p[3], p[4])};
  return qd_fused<true>(acc, pv);
}
#endif
MPSG_DI MC<3> fma_acc_d(const MC<3>& acc, const MC<3>& x, double a) {
  double p[4];
  td_mul_d_prenorm(x.c, a, p);
  const double ce[4] = {acc.c[0], acc.c[1], acc.c[2], 0.0};
  double t[5];
  qd_add_prenorm(ce, p, t);
  return renorm<3, 5>(t);
}
MPSG_DI MC<2> fma_acc_d(const MC<2>& acc, const MC<2>& x, double a) { return add(acc, mul_d(x, a)); }
// canonical form of a fma_acc accumulator before it is stored (once per row)
MPSG_DI MC<4> canon(const MC<4>& v) {
  double t[5] = {v.c[0], v.c[1], v.c[2], v.c[3], 0.0};
  return renorm<4, 5>(t);
}
MPSG_DI MC<3> canon(const MC<3>& v) {
#if MPSG_TD_SWEEP
  double t[4] = {v.c[0], v.c[1], v.c[2], 0.0};
  return renorm<3, 4>(t);
#else
  return v;
#endif
}
MPSG_DI MC<2> canon(const MC<2>& v) { return v; }

template <int K>
MPSG_DI MC<K> zero() {
  MC<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.c[i] = 0.0;
  return r;
}
template <int K>
MPSG_DI MC<K> from_double(double v) {  // MultiComponent(double), multicomp.hpp:23
  MC<K> r = zero<K>();
  r.c[0] = v;
  return r;
}
template <int K>
MPSG_DI MC<K> negate(const MC<K>& x) {  // multicomp.hpp:279-284
  MC<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.c[i] = -x.c[i];
  return r;
}
template <int K>
MPSG_DI MC<K> sub(const MC<K>& x, const MC<K>& y) {  // multicomp.hpp:286-289
  return add(x, negate(y));
}
// multicomp.hpp:291-302: K+1 quotient digits, then renorm<K>(q)
template <int K>
MPSG_DI MC<K> divide(const MC<K>& a, const MC<K>& b) {
  double q[K + 1];
  MC<K> r = a;
#pragma unroll
  for (int i = 0; i <= K; ++i) {
    q[i] = __ddiv_rn(r.c[0], b.c[0]);
    if (i < K) r = sub(r, mul_d(b, q[i]));
  }
  if constexpr (K == 2) {
    // renorm<2> = renorm_n<2,3>
    return renorm<2, 3>(q);
  } else {
    return renorm<K, K + 1>(q);
  }
}
// multicomp.hpp:304-322: Newton on 1/sqrt(a), then one multiply-back step
template <int K>
MPSG_DI MC<K> sqrt_mc(const MC<K>& a) {
  if (a.c[0] == 0.0) return zero<K>();
  if (a.c[0] < 0.0 || a.c[0] != a.c[0]) return from_double<K>(__longlong_as_double(0x7ff8000000000000ll));
  MC<K> x = from_double<K>(__ddiv_rn(1.0, __dsqrt_rn(a.c[0])));
  const MC<K> one = from_double<K>(1.0);
  const int iters = (K == 4) ? 3 : 2;
  for (int i = 0; i < iters; ++i) {
    MC<K> e = sub(one, mul(a, mul(x, x)));
    x = add(x, mul_d(mul(x, e), 0.5));
  }
  MC<K> r = mul(a, x);
  r = add(r, mul_d(mul(sub(a, mul(r, r)), x), 0.5));
  return r;
}
// multicomp.hpp:329-335
template <int K>
MPSG_DI double to_double(const MC<K>& x) {
  double s = x.c[K - 1];
#pragma unroll
  for (int i = K - 2; i >= 0; --i) s = dadd(x.c[i], s);
  return s;
}
// multicomp.hpp:342-351 (-2 when unordered)
template <int K>
MPSG_DI int compare(const MC<K>& x, const MC<K>& y) {
  if (x.c[0] != x.c[0] || y.c[0] != y.c[0]) return -2;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (x.c[i] < y.c[i]) return -1;
    if (x.c[i] > y.c[i]) return 1;
  }
  return 0;
}
template <int K>
MPSG_DI bool less_equal(const MC<K>& x, const MC<K>& y) {  // multicomp.hpp:390-393
  int c = compare(x, y);
  return c == 0 || c == -1;
}

// record_step's tests on ||r|| = sqrt(d) without the multi-component square
// root, when the outcome is certain: d's leading part is a normal positive
// double, and sqrt(d0) clears the threshold and stays under the divergence cap
// by a relative margin of 1e-9 (sqrt_mc(d) and sqrt(d0) agree to ~1e-16
// relative, as do thr and to_double(thr)).  Then rnorm > thr, rnorm is finite
// and to_double(rnorm) <= cap, i.e. the iteration continues -- the decision the
// exact test takes -- and the history entry to_double(sqrt_mc(d)) can be
// computed later, off the critical path of the solve.
template <int K>
MPSG_DI bool surely_continues(const MC<K>& d, const MC<K>& thr, double cap) {
  const double d0 = d.c[0];
  if (!(d0 >= 2.2250738585072014e-308 && d0 <= 1e300)) return false;  // also rejects NaN
  const double est = __dsqrt_rn(d0);
  return est > to_double(thr) * (1.0 + 1e-9) && est < cap * (1.0 - 1e-9);
}

// -------------------------------------------------------- memory helpers --
// L2 eviction-priority hints (createpolicy + ld.global.L2::cache_hint): the
// gathered vector x is loaded evict_last so the streamed matrix (evict_first)
// does not push it out of L2.  MPSG_X_HINT / MPSG_A_HINT select them.
#ifndef MPSG_X_HINT
#define MPSG_X_HINT 0
#endif
#ifndef MPSG_A_HINT
#define MPSG_A_HINT 0
#endif
MPSG_DI uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
MPSG_DI uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
MPSG_DI double2 ld_v2_hint(const double* q, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(q), "l"(pol));
  return r;
}
MPSG_DI double ld_f64_hint(const double* q, uint64_t pol) {
  double r;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(q), "l"(pol));
  return r;
}
MPSG_DI double ld_f64_stream(const double* q) {
#if MPSG_A_HINT
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(r)
               : "l"(q), "l"(policy_evict_first()));
  return r;
#else
  return __ldcs(q);
#endif
}
MPSG_DI int ld_s32_stream(const int* q) {
#if MPSG_A_HINT
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(r)
               : "l"(q), "l"(policy_evict_first()));
  return r;
#else
  return __ldcs(q);
#endif
}

// 256-bit x gathers: 0 ld.global.nc (L1-allocating), 1 ld.global.cg, 2 nc with
// L1::no_allocate, 3 nc with L1::evict_last.  Random gathers find almost nothing
// in L1 (1% hit rate in ncu), so not allocating is the default: cfg2 TD 195.6 ->
// 189.5 us (three alternating runs), QD and cfg5 unchanged.
#ifndef MPSG_X_LD
#define MPSG_X_LD 2
#endif
MPSG_DI void ld_v4(const double* q, double& a, double& b, double& c, double& d) {
#if MPSG_X_LD == 1
  asm("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(q));
#elif MPSG_X_LD == 2
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(q));
#elif MPSG_X_LD == 3
  asm("ld.global.nc.L1::evict_last.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(q));
#else
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(q));
#endif
}
// QD gather of x[i] as one 256-bit load (LDG.E.ENL2.256, sm_100; the caller
// guarantees p is 32-byte aligned) instead of two 128-bit ones: one L1
// wavefront per random gather instead of two.  The x gathers dominate the L1
// request load of the real SELL kernels (cfg2 QD ncu: L1/TEX 81% -> 57% busy,
// +2.3%).  A TD variant (the 24-byte element read from its aligned 32-byte
// window, or from two windows when it straddles) measured slower than three
// 64-bit loads (cfg2 TD 126.0 -> 123.0 Gnnz/s) and was dropped.
template <int K>
MPSG_DI MC<K> load_x_wide(const double* __restrict__ p, int64_t i) {
  static_assert(K == 4 || K == 3, "256-bit gathers: QD, and TD from the padded copy of x ([n][4])");
  MC<K> r;
  if constexpr (K == 4) {
    ld_v4(p + 4 * i, r.c[0], r.c[1], r.c[2], r.c[3]);
  } else {
    double pad;
    ld_v4(p + 4 * i, r.c[0], r.c[1], r.c[2], pad);
  }
  return r;
}

template <int K>
MPSG_DI MC<K> load_aos(const double* __restrict__ p, int64_t i) {
  MC<K> r;
  const double* q = p + i * K;
#if MPSG_X_HINT
  const uint64_t pol = policy_evict_last();
  if constexpr (K == 2 || K == 4) {
#pragma unroll
    for (int h = 0; h < K / 2; ++h) {
      double2 v = ld_v2_hint(q + 2 * h, pol);
      r.c[2 * h] = v.x;
      r.c[2 * h + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) r.c[j] = ld_f64_hint(q + j, pol);
  }
  return r;
#endif
  if constexpr (K == 2) {
    double2 v = __ldg(reinterpret_cast<const double2*>(q));
    r.c[0] = v.x;
    r.c[1] = v.y;
  } else if constexpr (K == 4) {
    double2 v0 = __ldg(reinterpret_cast<const double2*>(q));
    double2 v1 = __ldg(reinterpret_cast<const double2*>(q) + 1);
    r.c[0] = v0.x;
    r.c[1] = v0.y;
    r.c[2] = v1.x;
    r.c[3] = v1.y;
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) r.c[j] = __ldg(q + j);
  }
  return r;
}
// Plain (coherent) loads for vectors written earlier in the same launch
// sequence without a kernel boundary guarantee of read-only-ness.
template <int K>
MPSG_DI MC<K> load_aos_rw(const double* p, int64_t i) {
  MC<K> r;
#pragma unroll
  for (int j = 0; j < K; ++j) r.c[j] = p[i * K + j];
  return r;
}
template <int K>
MPSG_DI void store_aos(double* __restrict__ p, int64_t i, const MC<K>& v) {
  double* q = p + i * K;
  if constexpr (K == 2) {
    *reinterpret_cast<double2*>(q) = make_double2(v.c[0], v.c[1]);
  } else if constexpr (K == 4) {
    reinterpret_cast<double2*>(q)[0] = make_double2(v.c[0], v.c[1]);
    reinterpret_cast<double2*>(q)[1] = make_double2(v.c[2], v.c[3]);
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) q[j] = v.c[j];
  }
}
template <int K>
MPSG_DI MC<K> shfl_xor(const MC<K>& v, int mask) {
  MC<K> r;
#pragma unroll
  for (int j = 0; j < K; ++j) r.c[j] = __shfl_xor_sync(0xffffffffu, v.c[j], mask);
  return r;
}
template <int K>
MPSG_DI MC<K> shfl(const MC<K>& v, int src, unsigned mask = 0xffffffffu) {
  MC<K> r;
#pragma unroll
  for (int j = 0; j < K; ++j) r.c[j] = __shfl_sync(mask, v.c[j], src);
  return r;
}

// The scalar tails of the solve() engine's reductions (krylov_kernels.cuh) run
// once per launch on one thread, so their code is cold in the instruction
// cache every time: for QD the multi-component divide / sqrt are called, not
// inlined, and the warp tree is a loop (one copy of the add instead of five),
// which keeps those kernels a fraction of their inlined size: cfg5 QD ms /
// iteration BiCGSTAB 0.735 -> 0.685, GPBiCG 1.154 -> 1.070, CGS 0.596 -> 0.573
// (MPSG_CG_SMALL_TAIL=0 restores the inlined form).
#ifndef MPSG_CG_SMALL_TAIL
#define MPSG_CG_SMALL_TAIL 1
#endif
template <int K>
__device__ __noinline__ MC<K> divide_noinline(const MC<K>& a, const MC<K>& b) {
  return divide(a, b);
}
template <int K>
__device__ __noinline__ MC<K> sqrt_noinline(const MC<K>& a) {
  return sqrt_mc(a);
}
// QD only: the DD / TD tails are short
template <int K>
MPSG_DI MC<K> divide_call(const MC<K>& a, const MC<K>& b) {
  if constexpr (K == 4 && MPSG_CG_SMALL_TAIL)
    return divide_noinline(a, b);
  else
    return divide(a, b);
}
template <int K>
MPSG_DI MC<K> sqrt_call(const MC<K>& a) {
  if constexpr (K == 4 && MPSG_CG_SMALL_TAIL)
    return sqrt_noinline(a);
  else
    return sqrt_mc(a);
}
template <int K>
MPSG_DI MC<K> warp_tree(MC<K> v) {
  if constexpr (K == 4 && MPSG_CG_SMALL_TAIL) {
#pragma unroll 1
    for (int off = 16; off >= 1; off >>= 1) v = add(v, shfl_xor(v, off));
  } else {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = add(v, shfl_xor(v, off));
  }
  return v;
}

// Load-grouping helpers (spmv_kernels.cuh, MPSG_TIE): w accumulates the xor
// of one word of every loaded value; tie_apply xors it into a word of the
// first operand TWICE (identity), through opaque asm so that neither NVVM nor
// ptxas cancels it -- the first use of that operand then depends on every load.
MPSG_DI uint32_t tie_word(uint32_t w, double v) {
  uint32_t r;
  asm("xor.b32 %0, %1, %2;" : "=r"(r) : "r"(w), "r"((uint32_t)__double2loint(v)));
  return r;
}
MPSG_DI double tie_apply(double v, uint32_t w) {
  uint32_t lo = (uint32_t)__double2loint(v), t;
  asm("xor.b32 %0, %1, %2;" : "=r"(t) : "r"(lo), "r"(w));
  asm("xor.b32 %0, %1, %2;" : "=r"(lo) : "r"(t), "r"(w));
  return __hiloint2double(__double2hiint(v), (int)lo);
}

}  // namespace mpsg
