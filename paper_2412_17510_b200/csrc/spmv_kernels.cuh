// spmv_kernels.cuh -- sm_100a CSR SpMV kernels for DD/TD/QD, real and complex.
//
// Accumulation orders (the reference's, kernels.hpp):
//   ORDER_SCALAR  lanes off, row_sum_scalar (kernels.hpp:90-99):
//                 acc = +0; acc = acc + term(a_k, x[col_k]) for k in row order.
//   ORDER_LANE4   lanes on (the reference default, kernels.hpp:44),
//                 row_sum_lanes_pure/_mixed (kernels.hpp:103-142): lane j of 4
//                 takes k = b + 4m + j over whole groups,
//                 s = ((0+L0)+L1)+L2, s+L3, then the remainder appended serially.
// Both are reproduced bit-for-bit (mc_arith.cuh restates the op chains).
// The product term follows mul_term (kernels.hpp:50-60): Pure mode (matrix in
// MultiComponent<K>) is mul(a, v), matrix operand first; Mixed mode (binary64
// matrix, the paper's "M") is mul_by_double(v, a).  Template flag MX.
// Complex (kernels.hpp:399-416): rr = A.re x.re, ii = A.im x.im,
// ri = A.re x.im, ir = A.im x.re, each a full row sum in the chosen order,
// then y.re = rr - ii, y.im = ri + ir -- fused into one pass over A and x.
// With CONJ (the adjoint of sptmv_complex, kernels.hpp:419-441, run on the
// transposed matrix) the combine is y.re = rr + ii, y.im = ri - ir.
//
// Fast mode (ORDER_FAST) walks short rows in the lanes-off element order with
// the fused product-accumulate (fma_acc, one renormalisation sweep per
// nonzero) and cuts long rows into warp chunks: lanes accumulate strided
// partials, a fixed shuffle tree and a fixed chunk-order combine finish the
// row (deterministic, but not the reference's bits; checked against the
// componentwise bound).
#pragma once

#include <type_traits>

#include "layout.h"
#include "mc_arith.cuh"

namespace mpsg {

enum { ORDER_SCALAR = 0, ORDER_LANE4 = 1, ORDER_FAST = 2 };

template <int K>
MPSG_DI MC<K> load_planes(const double* __restrict__ val, int64_t stride, int64_t e) {
  MC<K> a;
#pragma unroll
  for (int j = 0; j < K; ++j) a.c[j] = __ldg(val + j * stride + e);
  return a;
}

// Streamed (evict-first) variant for matrix data that is read exactly once.
template <int K>
MPSG_DI MC<K> load_planes_stream(const double* __restrict__ val, int64_t stride, int64_t e) {
  MC<K> a;
#pragma unroll
  for (int j = 0; j < K; ++j) a.c[j] = ld_f64_stream(val + j * stride + e);
  return a;
}

// One matrix element and its product with a vector element (mul_term,
// kernels.hpp:50-60).  NPL = value planes per (re / im) part of the matrix.
template <int K, bool MX>
struct AVal;
template <int K>
struct AVal<K, false> {  // Pure: K component planes, mul(a, v)
  static constexpr int NPL = K;
  MC<K> a;
  MPSG_DI void load(const double* __restrict__ vp, int64_t st, int64_t e) { a = load_planes_stream<K>(vp, st, e); }
  MPSG_DI void load_ldg(const double* __restrict__ vp, int64_t st, int64_t e) { a = load_planes<K>(vp, st, e); }
  MPSG_DI MC<K> times(const MC<K>& v) const { return mul(a, v); }
  // FAST order: acc + a*v with one renormalisation (mc_arith.cuh fma_fast)
  MPSG_DI MC<K> accumulate(const MC<K>& acc, const MC<K>& v) const { return fma_acc(acc, a, v); }
  // TD/QD: into unnormalised level sums (fma_lvl, swept per group by the caller)
  MPSG_DI void accumulate_lvl(MC<K>& acc, const MC<K>& v) const {
    if constexpr (K >= 3)
      fma_lvl(acc, a, v);
    else
      acc = fma_acc(acc, a, v);
  }
};
template <int K>
struct AVal<K, true> {  // Mixed: one binary64 plane, mul_by_double(v, a)
  static constexpr int NPL = 1;
  double a;
  MPSG_DI void load(const double* __restrict__ vp, int64_t, int64_t e) { a = ld_f64_stream(vp + e); }
  MPSG_DI void load_ldg(const double* __restrict__ vp, int64_t, int64_t e) { a = __ldg(vp + e); }
  MPSG_DI MC<K> times(const MC<K>& v) const { return mul_d(v, a); }
  MPSG_DI MC<K> accumulate(const MC<K>& acc, const MC<K>& v) const { return fma_acc_d(acc, v, a); }
  MPSG_DI void accumulate_lvl(MC<K>& acc, const MC<K>& v) const {
    if constexpr (K >= 3)
      fma_lvl_d(acc, v, a);
    else
      acc = fma_acc_d(acc, v, a);
  }
};

// ---------------------------------------------------------------------------
// Row-sum building blocks for the SELL kernels (slot stride 32).
// ---------------------------------------------------------------------------
// 8 resident blocks of 128 threads (64 registers): measured +4-7% on the FAST
// TD/QD short-row kernels (profiles/r01b_variants.txt, item 36); MPSG_SELL_MINB=0
// removes the cap.
#ifndef MPSG_SELL_MINB
#define MPSG_SELL_MINB 8
#endif
// TD/QD only: DD (memory-latency-bound) keeps the compiler's own allocation --
// minBlocks 0 compiles to the same SASS as no bound (40 registers, 32 in Mixed
// mode); a 64 cap let it grow (cfg5 DD 228 -> 197 Gnnz/s) and a 12-block cap
// changed its schedule (-6%).
// TD with the level accumulators: 7 resident blocks (72 registers, no spills)
// beat 8 (cfg2 TD 222 -> 196 us, cfg5 TD 103 -> 97 us); QD keeps 8 (72
// registers: cfg2 QD 292 -> 325 us).
#ifndef MPSG_SELL_MINB_TD
#define MPSG_SELL_MINB_TD 7
#endif
#if MPSG_SELL_MINB > 0
#define MPSG_SELL_LB \
  __launch_bounds__(128, (K == 2 ? 0 : (K == 3 && ORDER == ORDER_FAST ? MPSG_SELL_MINB_TD : MPSG_SELL_MINB)))
#else
#define MPSG_SELL_LB __launch_bounds__(128)
#endif

// Products per round of the FAST QD short-row chain.  With the level-wise
// accumulate (121 ops) the QD kernel is latency-limited: four products in
// flight under a 64-register cap (MPSG_SELL_MINB 8) beat two (cfg2 QD 91.1 ->
// 99.8 Gnnz/s); TD (52 ops) keeps two (G = 4 for TD: 126.3 -> 122.1).
#ifndef MPSG_CPLX_TIE_L4
#define MPSG_CPLX_TIE_L4 2
#endif
#ifndef MPSG_CPLX_TIE
#define MPSG_CPLX_TIE 5
#endif
#ifndef MPSG_DD_TAIL_TIE
#define MPSG_DD_TAIL_TIE 1
#endif
#ifndef MPSG_DD_L4_MINB
#define MPSG_DD_L4_MINB 10
#endif
#ifndef MPSG_DD_L4_TAIL_TIE
#define MPSG_DD_L4_TAIL_TIE 1
#endif
#ifndef MPSG_FUSED_G_QD
#define MPSG_FUSED_G_QD 4
#endif
#ifndef MPSG_FUSED_G_TD
#define MPSG_FUSED_G_TD 2
#endif
// FAST short rows: the products of a round go into unnormalised level sums
// (fma_lvl) and the backward sweep runs once per round instead of once per
// product (mc_arith.cuh).
#ifndef MPSG_LVL_ACC
#define MPSG_LVL_ACC 1
#endif

// x gather in the real SELL kernels: QD with one 256-bit load when x is
// 32-byte aligned (the kernel's XW flag, checked per launch), else the plain
// AoS loads.
template <int K>
MPSG_DI MC<K> load_x(const double* __restrict__ x, bool xw, int64_t i) {
  if constexpr (K == 4 || K == 3) {
    if (xw) return load_x_wide<K>(x, i);  // TD: x is the padded copy
  }
  return load_aos<K>(x, i);
}

// TD x [n][3] -> [n][4] (see mpsg_csr::xpad): four consecutive elements are
// three 256-bit loads and four 256-bit stores per thread.
static __global__ void __launch_bounds__(256) pad_td_kernel(const double* __restrict__ x, double* __restrict__ xp, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = __ldg(x + 3 * i), b = __ldg(x + 3 * i + 1), c = __ldg(x + 3 * i + 2);
  double4 v = make_double4(a, b, c, 0.0);
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(xp + 4 * i), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
               : "memory");
}

// Product term of slot-row element k.
template <int K, bool MX>
MPSG_DI MC<K> sell_term(const double* __restrict__ vp, const int* __restrict__ cp, int64_t st,
                        const double* __restrict__ x, bool xw, int k) {
  const int64_t e = (int64_t)k * 32;
  AVal<K, MX> a;
  a.load(vp, st, e);
  return a.times(load_x<K>(x, xw, ld_s32_stream(cp + e)));
}

// LANE4 order with the four lane chains evaluated P at a time.  Chain j
// accumulates elements j, j+4, ... of the row's whole 4-groups; the lane
// combine s = (((0 + L0) + L1) + L2) + L3 is folded in as soon as a chain is
// complete, which is the reference's order (kernels.hpp:108-115) -- only the
// schedule differs, so fewer accumulators are live at once (P*K doubles
// instead of 4*K) and more warps fit per SM.  P = 2 for DD (latency-bound:
// more loads in flight), 1 for TD/QD (fp64-bound: fewer registers);
// measured in profiles/r01b_variants.txt.
template <int K, bool MX>
MPSG_DI MC<K> lane4_row(const double* __restrict__ vp, const int* __restrict__ cp, int64_t st,
                        const double* __restrict__ x, bool xw, int len) {
  constexpr int P = K == 2 ? 2 : 1;
  const int nfull = len >> 2;
  MC<K> s = zero<K>();
#pragma unroll
  for (int j0 = 0; j0 < 4; j0 += P) {
    MC<K> L[P];
#pragma unroll
    for (int c = 0; c < P; ++c) L[c] = zero<K>();
    if constexpr (P == 1) {
      // one chain: the next element's column index is loaded a round ahead
      int c = nfull > 0 ? ld_s32_stream(cp + (int64_t)j0 * 32) : 0;
      for (int m = 0; m < nfull; ++m) {
        const int e = 4 * m + j0;
        const int cn = (m + 1 < nfull) ? ld_s32_stream(cp + (int64_t)(e + 4) * 32) : 0;
        AVal<K, MX> a;
        a.load(vp, st, (int64_t)e * 32);
        L[0] = add(L[0], a.times(load_x<K>(x, xw, c)));
        c = cn;
      }
    } else {
      for (int m = 0; m < nfull; ++m) {
#pragma unroll
        for (int c = 0; c < P; ++c) L[c] = add(L[c], sell_term<K, MX>(vp, cp, st, x, xw, 4 * m + j0 + c));
      }
    }
#pragma unroll
    for (int c = 0; c < P; ++c) s = add(s, L[c]);
  }
#if MPSG_DD_L4_TAIL_TIE
  if constexpr (K == 2 && !MX) {
    // the remainder (1-3 elements) as one tied group, as in scalar_row
    const int k0 = nfull * 4, rem = len - k0;
    if (rem == 1) {
      s = add(s, sell_term<K, MX>(vp, cp, st, x, xw, k0));
    } else if (rem > 1) {
      int c[3];
      AVal<K, MX> a[3];
      MC<K> v[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) c[j] = ld_s32_stream(cp + (int64_t)(k0 + min(j, rem - 1)) * 32);
#pragma unroll
      for (int j = 0; j < 3; ++j) a[j].load(vp, st, (int64_t)(k0 + min(j, rem - 1)) * 32);
#pragma unroll
      for (int j = 0; j < 3; ++j) v[j] = load_x<K>(x, xw, c[j]);
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        w = tie_word(w, a[j].a.c[0]);
        w = tie_word(w, a[j].a.c[1]);
        w = tie_word(w, v[j].c[0]);
      }
      a[0].a.c[0] = tie_apply(a[0].a.c[0], w);
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (j < rem) s = add(s, a[j].times(v[j]));
    }
    return s;
  }
#endif
  for (int k = nfull * 4; k < len; ++k) s = add(s, sell_term<K, MX>(vp, cp, st, x, xw, k));
  return s;
}

// Lanes-off order (row_sum_scalar, kernels.hpp:90-99): one serial chain.  The
// products of G consecutive elements are formed first (G gathers in flight),
// then added in order.  PF = 1 also loads the next group's column indices a
// round ahead, so its gathers issue as soon as the group starts.  DD: G = 4,
// no prefetch (occupancy-bound); TD/QD: G = 2 with prefetch (64 registers).
template <int K, bool MX, bool FUSED = false>
MPSG_DI MC<K> scalar_row(const double* __restrict__ vp, const int* __restrict__ cp, int64_t st,
                         const double* __restrict__ x, bool xw, int len) {
  constexpr int G = K == 2 ? 4 : (FUSED ? (K == 4 ? MPSG_FUSED_G_QD : MPSG_FUSED_G_TD) : 2);
  constexpr bool PF = K != 2;
  MC<K> acc = zero<K>();
  int k = 0;
  if constexpr (PF) {
    int c[G];
#pragma unroll
    for (int j = 0; j < G; ++j) c[j] = (j < len) ? ld_s32_stream(cp + (int64_t)j * 32) : 0;
    for (; k + G <= len; k += G) {
      int cn[G];
#pragma unroll
      for (int j = 0; j < G; ++j) cn[j] = (k + G + j < len) ? ld_s32_stream(cp + (int64_t)(k + G + j) * 32) : 0;
      if constexpr (FUSED) {
        AVal<K, MX> a[G];
        MC<K> v[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          a[j].load(vp, st, (int64_t)(k + j) * 32);
          v[j] = load_x<K>(x, xw, c[j]);
        }
#if MPSG_LVL_ACC
#pragma unroll
        for (int j = 0; j < G; ++j) a[j].accumulate_lvl(acc, v[j]);
        acc = lvl_sweep(acc);
#else
#pragma unroll
        for (int j = 0; j < G; ++j) acc = a[j].accumulate(acc, v[j]);
#endif
      } else {
        MC<K> p[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          AVal<K, MX> a;
          a.load(vp, st, (int64_t)(k + j) * 32);
          p[j] = a.times(load_x<K>(x, xw, c[j]));
        }
#pragma unroll
        for (int j = 0; j < G; ++j) acc = add(acc, p[j]);
      }
#pragma unroll
      for (int j = 0; j < G; ++j) c[j] = cn[j];
    }
    // the tail's column indices are already in c[] (loaded a round ahead):
    // no dependent column load at the end of the row (TD/QD +1%, CG QD +1.7%)
#pragma unroll
    for (int j = 0; j < G - 1; ++j)
      if (k + j < len) {
        AVal<K, MX> a;
        a.load(vp, st, (int64_t)(k + j) * 32);
        if constexpr (FUSED) {
#if MPSG_LVL_ACC
          a.accumulate_lvl(acc, load_x<K>(x, xw, c[j]));
#else
          acc = a.accumulate(acc, load_x<K>(x, xw, c[j]));
#endif
        } else {
          acc = add(acc, a.times(load_x<K>(x, xw, c[j])));
        }
      }
#if MPSG_LVL_ACC
    if constexpr (FUSED) acc = lvl_sweep(acc);
#endif
    if constexpr (FUSED) acc = canon(acc);
    return acc;
  } else {
    for (; k + G <= len; k += G) {
      MC<K> p[G];
#pragma unroll
      for (int j = 0; j < G; ++j) p[j] = sell_term<K, MX>(vp, cp, st, x, xw, k + j);
#pragma unroll
      for (int j = 0; j < G; ++j) acc = add(acc, p[j]);
    }
#if MPSG_DD_TAIL_TIE
    if constexpr (K == 2 && !MX) {
      // the row's last 1..G-1 elements as one group: their columns, then their
      // value pairs and x gathers, in flight together (tie_word, mc_arith.cuh;
      // slots past the row's end repeat its last element and are not added)
      // instead of one element -- two dependent round trips -- at a time
      const int rem = len - k;
      if (rem == 1) {
        acc = add(acc, sell_term<K, MX>(vp, cp, st, x, xw, k));
      } else if (rem > 1) {
        int c[G - 1];
        AVal<K, MX> a[G - 1];
        MC<K> v[G - 1];
#pragma unroll
        for (int j = 0; j < G - 1; ++j) c[j] = ld_s32_stream(cp + (int64_t)(k + min(j, rem - 1)) * 32);
#pragma unroll
        for (int j = 0; j < G - 1; ++j) a[j].load(vp, st, (int64_t)(k + min(j, rem - 1)) * 32);
#pragma unroll
        for (int j = 0; j < G - 1; ++j) v[j] = load_x<K>(x, xw, c[j]);
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < G - 1; ++j) {
          w = tie_word(w, a[j].a.c[0]);
          w = tie_word(w, a[j].a.c[1]);
          w = tie_word(w, v[j].c[0]);
        }
        a[0].a.c[0] = tie_apply(a[0].a.c[0], w);
#pragma unroll
        for (int j = 0; j < G - 1; ++j)
          if (j < rem) acc = add(acc, a[j].times(v[j]));
      }
    } else
#endif
    {
      for (; k < len; ++k) acc = add(acc, sell_term<K, MX>(vp, cp, st, x, xw, k));
    }
    return acc;
  }
}

// Transposed product at T threads (kernels.hpp:368-394): the reference gives
// each of T row blocks (partition_rows) its own zero accumulator and merges
// them in thread order, y = acc_0, then y = y + acc_t for t = 1..T-1 -- for
// every output, touched or not.  On A^T (row j = column j of A, entries in
// ascending original row i) that is a fold over the T segments of row j cut at
// bounds[t]: each segment summed from zero in row order, the segment sums
// added in order.  `SegFold` walks one row's entries and does exactly that.
template <int K>
struct SegFold {
  const int64_t* bounds;
  int T, t;
  int64_t next;
  MC<K> y, acc;
  MPSG_DI SegFold(const int64_t* b, int T_) : bounds(b), T(T_), t(0), next(__ldg(b + 1)), y(zero<K>()), acc(zero<K>()) {}
  MPSG_DI void close() {
    if (t == 0)
      y = acc;
    else
      y = add(y, acc);
    acc = zero<K>();
    ++t;
    next = t < T ? __ldg(bounds + t + 1) : INT64_MAX;
  }
  MPSG_DI void push(int64_t i, const MC<K>& p) {  // entry of original row i
    while (i >= next) close();
    acc = add(acc, p);
  }
  MPSG_DI MC<K> finish() {
    while (t < T) close();
    return y;
  }
};

// ---------------------------------------------------------------------------
// SELL slice, real: one warp per slice of 32 rows, one thread per row.
// ---------------------------------------------------------------------------
// Row sum of slot `lane` of SELL slice s in the chosen order; row = the
// original row (-1 for padding).
template <int K, int ORDER, bool MX, bool XW>
MPSG_DI MC<K> sell_row(const SellView& S, const double* __restrict__ x, int s, int lane, int& row) {
  const int slot = s * 32 + lane;
  row = S.slot_row[slot];
  const int len = S.slot_len[slot];
  const int64_t base = S.slice_ptr[s] + lane;
  const int* __restrict__ cp = S.col + base;
  const double* __restrict__ vp = S.val + base;
  constexpr bool xw = XW;
  if constexpr (ORDER == ORDER_SCALAR)
    return scalar_row<K, MX>(vp, cp, S.stride, x, xw, len);
  else if constexpr (ORDER == ORDER_FAST)
    return scalar_row<K, MX, true>(vp, cp, S.stride, x, xw, len);  // fused multiply-accumulate (TD/QD)
  else
    return lane4_row<K, MX>(vp, cp, S.stride, x, xw, len);
}

// XW: x is 32-byte aligned and gathered with 256-bit loads (load_x_wide);
// the launcher checks the alignment of each call's x.
template <int K, int ORDER, bool MX, bool XW>
MPSG_DI void sell_real_body(const SellView& S, const double* __restrict__ x, double* __restrict__ y) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= S.nslices) return;
  int row;
  const MC<K> acc = sell_row<K, ORDER, MX, XW>(S, x, s, threadIdx.x & 31, row);
  if (row >= 0) store_aos<K>(y, row, acc);
}

template <int K, int ORDER, bool MX, bool XW>
__global__ void MPSG_SELL_LB sell_real_kernel(SellView S, const double* __restrict__ x, double* __restrict__ y) {
  sell_real_body<K, ORDER, MX, XW>(S, x, y);
}
// DD in the LANE4 order is memory-latency-bound: a resident-block floor (12
// blocks / 40 registers measured +17% on config 5 in round 1; 10 blocks / 48
// registers with the tied remainder group, round 2: cfg5 DD LANE4 71.7 -> 67.6 us).
template <int K, bool MX>
__global__ void __launch_bounds__(128, MPSG_DD_L4_MINB) sell_real_lane4_lat_kernel(SellView S, const double* __restrict__ x,
                                                                     double* __restrict__ y) {
  sell_real_body<K, ORDER_LANE4, MX, false>(S, x, y);
}

// Transposed product at T > 1 threads, real (see SegFold).
template <int K, bool MX>
__global__ void __launch_bounds__(128) sell_real_seg_kernel(SellView S, const double* __restrict__ x,
                                                            double* __restrict__ y, const int64_t* segb, int segT) {
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= S.nslices) return;
  const int slot = s * 32 + lane;
  const int row = S.slot_row[slot];
  const int len = S.slot_len[slot];
  const int64_t base = S.slice_ptr[s] + lane;
  SegFold<K> f(segb, segT);
  for (int k = 0; k < len; ++k) {
    const int64_t e = base + (int64_t)k * 32;
    const int c = ld_s32_stream(S.col + e);
    AVal<K, MX> a;
    a.load(S.val, S.stride, e);
    f.push(c, a.times(load_aos<K>(x, c)));
  }
  const MC<K> r = f.finish();
  if (row >= 0) store_aos<K>(y, row, r);
}

// ---------------------------------------------------------------------------
// SELL slice, complex: one warp per slice of 16 rows, two threads per row.
// Lanes 0-15 ("re" half) own rr = A.re x.re and ri = A.re x.im; lanes 16-31
// ("im" half) own ii = A.im x.im and ir = A.im x.re.  Each sum is its own
// chain in the chosen order; the combine happens in the re half.
// ---------------------------------------------------------------------------
template <int K, bool CONJ>
MPSG_DI void complex_store(double* __restrict__ yre, double* __restrict__ yim, int row, const MC<K>& rr,
                           const MC<K>& ii, const MC<K>& ri, const MC<K>& ir) {
  if constexpr (CONJ) {
    store_aos<K>(yre, row, add(rr, ii));  // rr + ii
    store_aos<K>(yim, row, sub(ri, ir));  // ri - ir
  } else {
    store_aos<K>(yre, row, sub(rr, ii));  // rr - ii
    store_aos<K>(yim, row, add(ri, ir));  // ri + ir
  }
}

template <int K, int ORDER, bool MX, bool CONJ, bool SEG = false>
__global__ void __launch_bounds__(128) sell_complex_kernel(SellView S, const double* __restrict__ xre,
                                                           const double* __restrict__ xim,
                                                           double* __restrict__ yre,
                                                           double* __restrict__ yim,
                                                           const int64_t* segb = nullptr, int segT = 1) {
  const int lane = threadIdx.x & 31;
  const int t = lane & 15;
  const bool imh = lane >= 16;
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= S.nslices) return;
  const int slot = s * 16 + t;
  const int row = S.slot_row[slot];
  const int len = S.slot_len[slot];
  const int64_t base = S.slice_ptr[s] + t;
  const int* __restrict__ cp = S.col + base;
  const int64_t st = S.stride;
  const double* __restrict__ vp = S.val + base + (imh ? (int64_t)AVal<K, MX>::NPL * st : 0);
  // first sum: re half rr (x.re), im half ii (x.im); second: ri (x.im), ir (x.re)
  const double* __restrict__ x1 = imh ? xim : xre;
  const double* __restrict__ x2 = imh ? xre : xim;

  MC<K> s1 = zero<K>(), s2 = zero<K>();
  if constexpr (SEG) {  // transposed product at T > 1 threads (SegFold), per sum
    SegFold<K> f1(segb, segT), f2(segb, segT);
    for (int k = 0; k < len; ++k) {
      const int64_t e = (int64_t)k * 16;
      const int c = ld_s32_stream(cp + e);
      AVal<K, MX> a;
      a.load(vp, st, e);
      f1.push(c, a.times(load_aos<K>(x1, c)));
      f2.push(c, a.times(load_aos<K>(x2, c)));
    }
    s1 = f1.finish();
    s2 = f2.finish();
  } else if constexpr ((ORDER == ORDER_SCALAR || ORDER == ORDER_FAST) && K == 2 && !MX && MPSG_CPLX_TIE > 1) {
    // DD (latency-bound): T elements per round, their column indices loaded a
    // round ahead and their value pairs and four x gathers forced into flight
    // together (tie_word, mc_arith.cuh); each sum still adds its terms in
    // element order -- the same bits as one element per round.
    constexpr int T = MPSG_CPLX_TIE;
    int c[T];
#pragma unroll
    for (int j = 0; j < T; ++j) c[j] = j < len ? ld_s32_stream(cp + (int64_t)j * 16) : 0;
    int k = 0;
    // one round of T elements from k; PARTIAL: the row's last round, whose
    // missing elements load the row's last one again (a valid address) and
    // are not accumulated
    auto round = [&](auto partial_tag) {
      constexpr bool PARTIAL = decltype(partial_tag)::value;
      int cn[T];
#pragma unroll
      for (int j = 0; j < T; ++j)
        cn[j] = (!PARTIAL && k + T + j < len) ? ld_s32_stream(cp + (int64_t)(k + T + j) * 16) : 0;
      AVal<K, MX> a[T];
      MC<K> v1[T], v2[T];
      const int last = PARTIAL ? len - 1 - k : T - 1;
#pragma unroll
      for (int j = 0; j < T; ++j) a[j].load(vp, st, (int64_t)(k + (PARTIAL ? min(j, last) : j)) * 16);
#pragma unroll
      for (int j = 0; j < T; ++j) {
        v1[j] = load_aos<K>(x1, c[j]);
        v2[j] = load_aos<K>(x2, c[j]);
      }
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < T; ++j) {
        w = tie_word(w, a[j].a.c[0]);
        w = tie_word(w, a[j].a.c[1]);
        w = tie_word(w, v1[j].c[0]);
        w = tie_word(w, v2[j].c[0]);
      }
      a[0].a.c[0] = tie_apply(a[0].a.c[0], w);
#pragma unroll
      for (int j = 0; j < T; ++j) {
        if (!PARTIAL || j <= last) {
          if constexpr (ORDER == ORDER_FAST) {
            s1 = a[j].accumulate(s1, v1[j]);
            s2 = a[j].accumulate(s2, v2[j]);
          } else {
            s1 = add(s1, a[j].times(v1[j]));
            s2 = add(s2, a[j].times(v2[j]));
          }
        }
      }
#pragma unroll
      for (int j = 0; j < T; ++j) c[j] = cn[j];
    };
    for (; k + T <= len; k += T) round(std::false_type{});
    if (k < len) round(std::true_type{});
  } else if constexpr (ORDER == ORDER_SCALAR || ORDER == ORDER_FAST) {
    int c = len > 0 ? ld_s32_stream(cp) : 0;  // column index loaded a round ahead
    for (int k = 0; k < len; ++k) {
      const int64_t e = (int64_t)k * 16;
      const int cn = (k + 1 < len) ? ld_s32_stream(cp + e + 16) : 0;
      AVal<K, MX> a;
      a.load(vp, st, e);
      if constexpr (ORDER == ORDER_FAST && !MX) {  // one renormalisation sweep per product-accumulate
        // (Pure mode: the level sums with a sweep per four products measured
        // slower here, cfg3 QD 29.6 -> 26.5 Gnnz/s: two accumulators per thread)
        s1 = a.accumulate(s1, load_aos<K>(x1, c));
        s2 = a.accumulate(s2, load_aos<K>(x2, c));
      } else if constexpr (ORDER == ORDER_FAST) {  // Mixed: level sums, one backward sweep per four products
        a.accumulate_lvl(s1, load_aos<K>(x1, c));
        a.accumulate_lvl(s2, load_aos<K>(x2, c));
        if ((k & 3) == 3 || k + 1 == len) {
          s1 = lvl_sweep(s1);
          s2 = lvl_sweep(s2);
        }
      } else {
        MC<K> p1 = a.times(load_aos<K>(x1, c));
        MC<K> p2 = a.times(load_aos<K>(x2, c));
        s1 = add(s1, p1);
        s2 = add(s2, p2);
      }
      c = cn;
    }
  } else {
    // the two sums' lane chains one at a time (reference order, fewer live
    // accumulators), see lane4_row
    const int nfull = len >> 2;
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      MC<K> L1 = zero<K>(), L2 = zero<K>();
      int m = 0;
      if constexpr (K == 2 && !MX && MPSG_CPLX_TIE_L4 > 1) {
        // DD: T elements of the chain per round, loads tied into flight
        // together (as the SCALAR / FAST branch above); same order, same bits
        constexpr int T = MPSG_CPLX_TIE_L4;
        for (; m + T <= nfull; m += T) {
          int c[T];
          AVal<K, MX> a[T];
          MC<K> v1[T], v2[T];
#pragma unroll
          for (int t = 0; t < T; ++t) c[t] = ld_s32_stream(cp + (int64_t)(4 * (m + t) + j) * 16);
#pragma unroll
          for (int t = 0; t < T; ++t) a[t].load(vp, st, (int64_t)(4 * (m + t) + j) * 16);
#pragma unroll
          for (int t = 0; t < T; ++t) {
            v1[t] = load_aos<K>(x1, c[t]);
            v2[t] = load_aos<K>(x2, c[t]);
          }
          uint32_t w = 0;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            w = tie_word(w, a[t].a.c[0]);
            w = tie_word(w, a[t].a.c[1]);
            w = tie_word(w, v1[t].c[0]);
            w = tie_word(w, v2[t].c[0]);
          }
          a[0].a.c[0] = tie_apply(a[0].a.c[0], w);
#pragma unroll
          for (int t = 0; t < T; ++t) {
            L1 = add(L1, a[t].times(v1[t]));
            L2 = add(L2, a[t].times(v2[t]));
          }
        }
      }
      for (; m < nfull; ++m) {
        const int64_t e = (int64_t)(4 * m + j) * 16;
        AVal<K, MX> a;
        a.load(vp, st, e);
        const int c = ld_s32_stream(cp + e);
        L1 = add(L1, a.times(load_aos<K>(x1, c)));
        L2 = add(L2, a.times(load_aos<K>(x2, c)));
      }
      s1 = add(s1, L1);
      s2 = add(s2, L2);
    }
    for (int k = nfull * 4; k < len; ++k) {
      const int64_t e = (int64_t)k * 16;
      AVal<K, MX> a;
      a.load(vp, st, e);
      const int c = ld_s32_stream(cp + e);
      s1 = add(s1, a.times(load_aos<K>(x1, c)));
      s2 = add(s2, a.times(load_aos<K>(x2, c)));
    }
  }
  // re half: s1 = rr, s2 = ri; im half: s1 = ii, s2 = ir
  MC<K> o1 = shfl(s1, lane ^ 16);
  MC<K> o2 = shfl(s2, lane ^ 16);
  if (!imh && row >= 0) complex_store<K, CONJ>(yre, yim, row, s1, o1, s2, o2);
}

// ---------------------------------------------------------------------------
// Long rows, deterministic: one CTA per row.  All threads form the products
// of a chunk into shared memory (they are independent); the reference's
// serial add chains then run on 1 (SCALAR) or 4 (LANE4) threads per sum.
// ---------------------------------------------------------------------------
template <int K, bool CPLX, bool MX>
MPSG_DI void long_products(const LongView& L, int64_t k, const double* __restrict__ xre,
                           const double* __restrict__ xim, MC<K>* out) {
  const int c = L.col[k];
  AVal<K, MX> are;
  are.load_ldg(L.val, L.stride, k);
  if constexpr (!CPLX) {
    out[0] = are.times(load_aos<K>(xre, c));
  } else {
    AVal<K, MX> aim;
    aim.load_ldg(L.val + (int64_t)AVal<K, MX>::NPL * L.stride, L.stride, k);
    MC<K> vr = load_aos<K>(xre, c), vi = load_aos<K>(xim, c);
    out[0] = are.times(vr);  // rr
    out[1] = aim.times(vi);  // ii
    out[2] = are.times(vi);  // ri
    out[3] = aim.times(vr);  // ir
  }
}

// Threads per CTA of the exact long-row kernel: the serial chains use 1 (SCALAR)
// or 4 (LANE4) threads of a CTA, so smaller CTAs put more chains on an SM.
#ifndef MPSG_LONG_DET_THREADS
#define MPSG_LONG_DET_THREADS 128
#endif
template <int K, int ORDER, bool CPLX, int CH, bool MX, bool CONJ, bool SEG = false>
__global__ void __launch_bounds__(MPSG_LONG_DET_THREADS) long_det_kernel(LongView L, const double* __restrict__ xre,
                                                       const double* __restrict__ xim,
                                                       double* __restrict__ yre,
                                                       double* __restrict__ yim,
                                                       const int64_t* segb = nullptr, int segT = 1) {
  constexpr int NS = CPLX ? 4 : 1;
  constexpr int NL = (ORDER == ORDER_LANE4) ? 4 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MC<K>* prod = reinterpret_cast<MC<K>*>(smem_raw);  // [CH][NS]

  const int r = blockIdx.x;
  const int64_t b = L.ptr[r];
  const int64_t len = L.ptr[r + 1] - b;
  const int64_t m4 = (ORDER == ORDER_LANE4) ? (len & ~int64_t(3)) : len;
  const int tid = threadIdx.x;
  // chain thread: sum = tid / NL, lane = tid % NL (tid < NS*NL)
  const bool chain = tid < NS * NL;
  const int sidx = tid / NL, lj = tid % NL;
  MC<K> acc = zero<K>();
  SegFold<K> fold(SEG ? segb : L.ptr, SEG ? segT : 1);  // SEG: transposed product at T > 1 threads
  int64_t c0 = 0;
  for (; c0 < len; c0 += CH) {
    const int cnt = (int)((len - c0) < CH ? (len - c0) : CH);
    constexpr int NT = MPSG_LONG_DET_THREADS;
    if constexpr (!CPLX && !MX && (CH % NT) == 0) {
      // a full chunk: this thread's CH / NT elements with their columns,
      // values and x gathers tied into flight together (tie_word,
      // mc_arith.cuh); the products are the same bits
      constexpr int E = CH / NT;
      if (cnt == CH) {
        int c[E];
        AVal<K, MX> a[E];
        MC<K> v[E];
#pragma unroll
        for (int u = 0; u < E; ++u) c[u] = L.col[b + c0 + tid + u * NT];
#pragma unroll
        for (int u = 0; u < E; ++u) a[u].load_ldg(L.val, L.stride, b + c0 + tid + u * NT);
#pragma unroll
        for (int u = 0; u < E; ++u) v[u] = load_aos<K>(xre, c[u]);
        uint32_t w = 0;
#pragma unroll
        for (int u = 0; u < E; ++u) {
#pragma unroll
          for (int q = 0; q < K; ++q) w = tie_word(w, a[u].a.c[q]);
          w = tie_word(w, v[u].c[0]);
          if constexpr (K > 2) w = tie_word(w, v[u].c[2]);
        }
        a[0].a.c[0] = tie_apply(a[0].a.c[0], w);
#pragma unroll
        for (int u = 0; u < E; ++u) prod[(tid + u * NT) * NS] = a[u].times(v[u]);
      } else {
        for (int i = tid; i < cnt; i += blockDim.x) long_products<K, CPLX, MX>(L, b + c0 + i, xre, xim, prod + i * NS);
      }
    } else {
      for (int i = tid; i < cnt; i += blockDim.x) long_products<K, CPLX, MX>(L, b + c0 + i, xre, xim, prod + i * NS);
    }
    __syncthreads();
    if (chain) {
      if constexpr (SEG) {
        for (int i = 0; i < cnt; ++i) fold.push(L.col[b + c0 + i], prod[i * NS + sidx]);
      } else {
        // this chain's products: i = first, first + step, ... below lim; four
        // shared-memory loads are tied into flight ahead of their four serial
        // adds (tie_word, mc_arith.cuh) -- same order, same bits
        constexpr int step = ORDER == ORDER_LANE4 ? 4 : 1;
        const int lim = ORDER == ORDER_LANE4 ? (int)((m4 - c0) < cnt ? (m4 - c0) : cnt) : cnt;
        int i = ORDER == ORDER_LANE4 ? lj : 0;
        for (; i + 3 * step < lim; i += 4 * step) {
          MC<K> q[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) q[u] = prod[(i + u * step) * NS + sidx];
          uint32_t w = 0;
#pragma unroll
          for (int u = 1; u < 4; ++u) w = tie_word(w, q[u].c[0]);
          q[0].c[0] = tie_apply(q[0].c[0], w);
#pragma unroll
          for (int u = 0; u < 4; ++u) acc = add(acc, q[u]);
        }
        for (; i < lim; i += step) acc = add(acc, prod[i * NS + sidx]);
      }
    }
    if (c0 + CH < len) __syncthreads();
  }
  c0 -= CH;  // start of the last chunk (still resident in shared memory)
  if constexpr (SEG) {
    if (chain) acc = fold.finish();
  }
  // all chain threads live in warp 0
  if (tid < 32) {
    MC<K> s = acc;
    if constexpr (ORDER == ORDER_LANE4) {
      MC<K> l1 = shfl(acc, (tid & ~3) + 1), l2 = shfl(acc, (tid & ~3) + 2), l3 = shfl(acc, (tid & ~3) + 3);
      s = add(add(add(add(zero<K>(), acc), l1), l2), l3);  // lanes 4*sidx hold L0
      if (chain && lj == 0)
        for (int64_t k = m4; k < len; ++k) s = add(s, prod[(k - c0) * NS + sidx]);
    }
    const int head = (ORDER == ORDER_LANE4) ? 4 : 1;  // lane stride between sums
    if constexpr (!CPLX) {
      if (tid == 0) store_aos<K>(yre, L.row[r], s);
    } else {
      MC<K> ii = shfl(s, 1 * head), ri = shfl(s, 2 * head), ir = shfl(s, 3 * head);
      if (tid == 0) complex_store<K, CONJ>(yre, yim, L.row[r], s, ii, ri, ir);
    }
  }
}

// ---------------------------------------------------------------------------
// Long rows, fast: one warp per chunk (see LongView: chunks are cut at
// column-block boundaries and issued block-major); lanes take strided
// elements (coalesced; real rows load the next column index a round ahead),
// a fixed xor-tree reduces the warp, and the last arriving warp of a row adds
// the chunk partials in row-position order.
// ---------------------------------------------------------------------------
template <int K, bool CPLX, bool MX, bool CONJ>
__global__ void __launch_bounds__(128) long_fast_kernel(LongView L, const double* __restrict__ xre,
                                                        const double* __restrict__ xim,
                                                        double* __restrict__ yre,
                                                        double* __restrict__ yim) {
  constexpr int NS = CPLX ? 4 : 1;
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= L.nchunks) return;
  const int r = L.chunk_row[w];
  const int first = L.chunk_first[r];
  const int nch = L.chunk_first[r + 1] - first;
  const int64_t b = L.chunk_beg[w];
  const int64_t e = L.chunk_end[w];

  MC<K> acc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) acc[s] = zero<K>();
  int64_t k = b + lane;
#ifndef MPSG_LONG_MX_U
#define MPSG_LONG_MX_U 4
#endif
#ifndef MPSG_LONG_U_DD
#define MPSG_LONG_U_DD 4
#endif
#ifndef MPSG_LONG_TIE
#define MPSG_LONG_TIE 1
#endif
  if constexpr (!CPLX) {
    // U elements per lane per round, accumulated in the lane's element order
    // (the same bits for every U).  ptxas keeps each load next to its use
    // whatever U is (40 registers for DD at U = 1..8, also with the loads in
    // one asm block); for DD the first accumulate of a round is therefore made
    // to depend on every load of the round (tie_word / tie_apply, an integer
    // xor identity), which puts the round's 4 gathers and 8 value loads in
    // flight together: cfg4 DD 587.8 -> 571.4 us.
    constexpr int U = MX ? MPSG_LONG_MX_U : (K == 2 ? MPSG_LONG_U_DD : 2);
    for (; k + 32 * (U - 1) < e; k += 32 * U) {
      int c[U];
      AVal<K, MX> a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = ld_s32_stream(L.col + k + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) a[u].load(L.val, L.stride, k + 32 * u);
      MC<K> v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = load_aos<K>(xre, c[u]);
#if MPSG_LONG_TIE
      if constexpr (K == 2) {
        // every load of the round in flight before the first accumulate (tie_word)
        uint32_t w = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if constexpr (MX) {
            w = tie_word(w, a[u].a);
          } else {
            w = tie_word(w, a[u].a.c[0]);
            w = tie_word(w, a[u].a.c[1]);
          }
          w = tie_word(w, v[u].c[0]);
        }
        if constexpr (MX)
          a[0].a = tie_apply(a[0].a, w);
        else
          a[0].a.c[0] = tie_apply(a[0].a.c[0], w);
      }
#endif
#pragma unroll
      for (int u = 0; u < U; ++u) a[u].accumulate_lvl(acc[0], v[u]);
      acc[0] = lvl_sweep(acc[0]);
    }
    for (; k < e; k += 32) {
      AVal<K, MX> a1;
      a1.load(L.val, L.stride, k);
      a1.accumulate_lvl(acc[0], load_aos<K>(xre, ld_s32_stream(L.col + k)));
      acc[0] = lvl_sweep(acc[0]);
    }
  } else {
    for (; k < e; k += 32) {
      const int c = ld_s32_stream(L.col + k);
      AVal<K, MX> are, aim;
      are.load(L.val, L.stride, k);
      aim.load(L.val + (int64_t)AVal<K, MX>::NPL * L.stride, L.stride, k);
      MC<K> vr = load_aos<K>(xre, c), vi = load_aos<K>(xim, c);
      are.accumulate_lvl(acc[0], vr);
      aim.accumulate_lvl(acc[1], vi);
      are.accumulate_lvl(acc[2], vi);
      aim.accumulate_lvl(acc[3], vr);
#pragma unroll
      for (int s = 0; s < NS; ++s) acc[s] = lvl_sweep(acc[s]);
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = add(acc[s], shfl_xor(acc[s], off));

  auto finish = [&](MC<K>* sums) {
    const int row = L.row[r];
    if constexpr (!CPLX)
      store_aos<K>(yre, row, sums[0]);
    else
      complex_store<K, CONJ>(yre, yim, row, sums[0], sums[1], sums[2], sums[3]);
  };
  if (nch == 1) {
    if (lane == 0) finish(acc);
    return;
  }
  double* part = L.partial + (int64_t)L.chunk_slot[w] * NS * K;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int j = 0; j < K; ++j) __stcg(part + s * K + j, acc[s].c[j]);
    __threadfence();
    const unsigned old = atomicAdd(L.counter + r, 1u);
    if (old == (unsigned)(nch - 1)) {
      __threadfence();
      MC<K> tot[NS];
      const double* p0 = L.partial + (int64_t)first * NS * K;
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int j = 0; j < K; ++j) tot[s].c[j] = __ldcg(p0 + s * K + j);
      for (int c = 1; c < nch; ++c) {
        const double* pc = p0 + (int64_t)c * NS * K;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          MC<K> v;
#pragma unroll
          for (int j = 0; j < K; ++j) v.c[j] = __ldcg(pc + s * K + j);
          tot[s] = add(tot[s], v);
        }
      }
      finish(tot);
      L.counter[r] = 0u;  // self-reset for the next launch
    }
  }
}

}  // namespace mpsg
