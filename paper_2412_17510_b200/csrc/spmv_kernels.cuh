// spmv_kernels.cuh -- sm_100a CSR SpMV kernels for DD/TD/QD, real and complex.
//
// Accumulation orders (the reference's, kernels.hpp):
//   ORDER_SCALAR  lanes off, row_sum_scalar (kernels.hpp:90-99):
//                 acc = +0; acc = acc + mul(a_k, x[col_k]) for k in row order.
//   ORDER_LANE4   lanes on (the reference default, kernels.hpp:44),
//                 row_sum_lanes_pure (kernels.hpp:103-121): lane j of 4 takes
//                 k = b + 4m + j over whole groups, s = ((0+L0)+L1)+L2, s+L3,
//                 then the remainder appended serially.
// Both are reproduced bit-for-bit (mc_arith.cuh restates the op chains).
// Complex (kernels.hpp:399-416): rr = A.re x.re, ii = A.im x.im,
// ri = A.re x.im, ir = A.im x.re, each a full row sum in the chosen order,
// then y.re = rr - ii, y.im = ri + ir -- fused into one pass over A and x.
//
// Fast mode (ORDER_FAST) differs only on long rows: a row is cut into
// warp-sized chunks, lanes accumulate strided partials with the reference
// ops, a fixed shuffle tree and a fixed chunk-order combine finish the row
// (deterministic, but not the reference order; checked against the
// componentwise bound).
#pragma once

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

// ---------------------------------------------------------------------------
// Row-sum building blocks for the SELL kernels.
// ---------------------------------------------------------------------------
// Lane chains evaluated concurrently in the LANE4 order (see lane4_row):
// 2 for DD (latency-bound: more loads in flight), 1 for TD/QD (fp64-bound:
// fewer live registers, more resident warps).  Measured on B200 in
// profiles/r01b_chain_variants.txt.
#ifndef MPSG_SELL_PAR_DD
#define MPSG_SELL_PAR_DD 2
#endif
#define MPSG_SELL_PAR(K) ((K) == 2 ? MPSG_SELL_PAR_DD : 1)
#ifdef MPSG_SELL_MINB
#define MPSG_SELL_LB __launch_bounds__(128, MPSG_SELL_MINB)
#else
#define MPSG_SELL_LB __launch_bounds__(128)
#endif

// One product term of slot-row element k (matrix operand first, kernels.hpp:52-54).
template <int K>
MPSG_DI MC<K> sell_term(const double* __restrict__ vp, const int* __restrict__ cp, int64_t st,
                        const double* __restrict__ x, int k) {
  const int64_t e = (int64_t)k * 32;
  return mul(load_planes_stream<K>(vp, st, e), load_aos<K>(x, ld_s32_stream(cp + e)));
}

// LANE4 order with the four lane chains evaluated P at a time.  Chain j
// accumulates elements j, j+4, ... of the row's whole 4-groups; the lane
// combine s = (((0 + L0) + L1) + L2) + L3 is folded in as soon as a chain is
// complete, which is the reference's order (kernels.hpp:108-115) -- only the
// schedule differs, so fewer accumulators are live at once (P*K doubles
// instead of 4*K) and more warps fit per SM.
template <int K, int P>
MPSG_DI MC<K> lane4_row(const double* __restrict__ vp, const int* __restrict__ cp, int64_t st,
                        const double* __restrict__ x, int len) {
  const int nfull = len >> 2;
  MC<K> s = zero<K>();
#pragma unroll
  for (int j0 = 0; j0 < 4; j0 += P) {
    MC<K> L[P];
#pragma unroll
    for (int c = 0; c < P; ++c) L[c] = zero<K>();
    if constexpr (P == 1 && K > 2) {
      // one chain: the next element's column index is loaded a round ahead
      int c = nfull > 0 ? ld_s32_stream(cp + (int64_t)j0 * 32) : 0;
      for (int m = 0; m < nfull; ++m) {
        const int e = 4 * m + j0;
        const int cn = (m + 1 < nfull) ? ld_s32_stream(cp + (int64_t)(e + 4) * 32) : 0;
        L[0] = add(L[0], mul(load_planes_stream<K>(vp, st, (int64_t)e * 32), load_aos<K>(x, c)));
        c = cn;
      }
    } else {
      for (int m = 0; m < nfull; ++m) {
#pragma unroll
        for (int c = 0; c < P; ++c) L[c] = add(L[c], sell_term<K>(vp, cp, st, x, 4 * m + j0 + c));
      }
    }
#pragma unroll
    for (int c = 0; c < P; ++c) s = add(s, L[c]);
  }
  for (int k = nfull * 4; k < len; ++k) s = add(s, sell_term<K>(vp, cp, st, x, k));
  return s;
}

// Chunked row sum for latency-bound (DD) rows.  The row is consumed CH
// elements at a time: first every column index of the chunk is loaded, then
// every gather and matrix value, so a thread has CH independent loads in
// flight per round trip instead of one; then the chunk's terms are added in
// the reference order -- lanes on: element k goes to chain k % 4 over whole
// 4-groups, chains combined (((0+L0)+L1)+L2)+L3, remainder serial; lanes off:
// one chain.  Indices past the row end are clamped to its last element (a
// valid address) and their terms discarded.
#ifndef MPSG_DD_CHUNK
#define MPSG_DD_CHUNK 0
#endif
template <int K, int ORDER, int CH>
MPSG_DI MC<K> chunked_row(const double* __restrict__ vp, const int* __restrict__ cp, int64_t st,
                          const double* __restrict__ x, int len) {
  constexpr bool LANES = ORDER != ORDER_SCALAR;
  const int body = LANES ? (len & ~3) : len;  // elements summed into the chains
  MC<K> L[LANES ? 4 : 1];
#pragma unroll
  for (int j = 0; j < (LANES ? 4 : 1); ++j) L[j] = zero<K>();
  auto load_chunk = [&](int k0, int lim, MC<K>* p) {
    int c[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = ld_s32_stream(cp + (int64_t)min(k0 + i, lim - 1) * 32);
    MC<K> xv[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) xv[i] = load_aos<K>(x, c[i]);
#pragma unroll
    for (int i = 0; i < CH; ++i) p[i] = mul(load_planes_stream<K>(vp, st, (int64_t)min(k0 + i, lim - 1) * 32), xv[i]);
  };
  MC<K> p[CH];
  int k0 = 0;
  if (len > 0) {
    for (;;) {  // the last chunk holds the (1..3 element) remainder, if any
      load_chunk(k0, len, p);
#pragma unroll
      for (int i = 0; i < CH; ++i)
        if (k0 + i < body) L[LANES ? (i & 3) : 0] = add(L[LANES ? (i & 3) : 0], p[i]);
      if (k0 + CH >= len) break;
      k0 += CH;
    }
  }
  MC<K> s;
  if constexpr (LANES) {
    s = zero<K>();
#pragma unroll
    for (int j = 0; j < 4; ++j) s = add(s, L[j]);
#pragma unroll
    for (int i = 0; i < CH; ++i)
      if (k0 + i >= body && k0 + i < len) s = add(s, p[i]);
  } else {
    s = L[0];
  }
  return s;
}

// Lanes-off order (row_sum_scalar, kernels.hpp:90-99): one serial chain.  The
// products of G consecutive elements are formed first (G gathers in flight),
// then added in order.  PF = 1 also loads the next group's column indices
// one round ahead, so its gathers can issue as soon as the group starts.
#ifndef MPSG_SCALAR_G
#define MPSG_SCALAR_G 2
#endif
#ifndef MPSG_SCALAR_PF
#define MPSG_SCALAR_PF 1
#endif
template <int K, int G, int PF>
MPSG_DI MC<K> scalar_row(const double* __restrict__ vp, const int* __restrict__ cp, int64_t st,
                         const double* __restrict__ x, int len) {
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
      MC<K> p[G];
#pragma unroll
      for (int j = 0; j < G; ++j)
        p[j] = mul(load_planes_stream<K>(vp, st, (int64_t)(k + j) * 32), load_aos<K>(x, c[j]));
#pragma unroll
      for (int j = 0; j < G; ++j) acc = add(acc, p[j]);
#pragma unroll
      for (int j = 0; j < G; ++j) c[j] = cn[j];
    }
  } else {
    for (; k + G <= len; k += G) {
      MC<K> p[G];
#pragma unroll
      for (int j = 0; j < G; ++j) p[j] = sell_term<K>(vp, cp, st, x, k + j);
#pragma unroll
      for (int j = 0; j < G; ++j) acc = add(acc, p[j]);
    }
  }
  for (; k < len; ++k) acc = add(acc, sell_term<K>(vp, cp, st, x, k));
  return acc;
}

// ---------------------------------------------------------------------------
// SELL slice, real: one warp per slice of 32 rows, one thread per row.
// ---------------------------------------------------------------------------
// Row sum of slot `lane` of SELL slice s in the chosen order; row = the
// original row (-1 for padding).
template <int K, int ORDER>
MPSG_DI MC<K> sell_row(const SellView& S, const double* __restrict__ x, int s, int lane, int& row) {
  const int slot = s * 32 + lane;
  row = S.slot_row[slot];
  const int len = S.slot_len[slot];
  const int64_t base = S.slice_ptr[s] + lane;
  const int* __restrict__ cp = S.col + base;
  const double* __restrict__ vp = S.val + base;
  const int64_t st = S.stride;

  MC<K> acc;
  if constexpr (K == 2 && MPSG_DD_CHUNK > 0) {
    acc = chunked_row<K, ORDER, MPSG_DD_CHUNK>(vp, cp, st, x, len);
  } else if constexpr (ORDER == ORDER_SCALAR) {
    acc = scalar_row<K, (K == 2 ? 4 : MPSG_SCALAR_G), (K == 2 ? 0 : MPSG_SCALAR_PF)>(vp, cp, st, x, len);
  } else {
    acc = lane4_row<K, MPSG_SELL_PAR(K)>(vp, cp, st, x, len);
  }
  return acc;
}

template <int K, int ORDER>
MPSG_DI void sell_real_body(const SellView& S, const double* __restrict__ x, double* __restrict__ y) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= S.nslices) return;
  int row;
  const MC<K> acc = sell_row<K, ORDER>(S, x, s, threadIdx.x & 31, row);
  if (row >= 0) store_aos<K>(y, row, acc);
}

template <int K, int ORDER>
__global__ void MPSG_SELL_LB sell_real_kernel(SellView S, const double* __restrict__ x, double* __restrict__ y) {
  sell_real_body<K, ORDER>(S, x, y);
}
// DD in the LANE4 order is memory-latency-bound: capped at 40 registers for
// 12 resident blocks per SM (measured +17% on config 5, profiles/r01b_*).
template <int K>
__global__ void __launch_bounds__(128, 12) sell_real_lane4_lat_kernel(SellView S, const double* __restrict__ x,
                                                                     double* __restrict__ y) {
  sell_real_body<K, ORDER_LANE4>(S, x, y);
}

// ---------------------------------------------------------------------------
// SELL slice, complex: one warp per slice of 16 rows, two threads per row.
// Lanes 0-15 ("re" half) own rr = A.re x.re and ri = A.re x.im; lanes 16-31
// ("im" half) own ii = A.im x.im and ir = A.im x.re.  Each sum is its own
// chain in the chosen order; the combine happens in the re half.
// ---------------------------------------------------------------------------
template <int K, int ORDER>
__global__ void __launch_bounds__(128) sell_complex_kernel(SellView S, const double* __restrict__ xre,
                                                           const double* __restrict__ xim,
                                                           double* __restrict__ yre,
                                                           double* __restrict__ yim) {
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
  const double* __restrict__ vp = S.val + base + (imh ? (int64_t)K * st : 0);
  // first sum: re half rr (x.re), im half ii (x.im); second: ri (x.im), ir (x.re)
  const double* __restrict__ x1 = imh ? xim : xre;
  const double* __restrict__ x2 = imh ? xre : xim;

  MC<K> s1 = zero<K>(), s2 = zero<K>();
  if constexpr (ORDER == ORDER_SCALAR) {
    int c = len > 0 ? ld_s32_stream(cp) : 0;  // column index loaded a round ahead
    for (int k = 0; k < len; ++k) {
      const int64_t e = (int64_t)k * 16;
      const int cn = (k + 1 < len) ? ld_s32_stream(cp + e + 16) : 0;
      MC<K> a = load_planes_stream<K>(vp, st, e);
      MC<K> p1 = mul(a, load_aos<K>(x1, c));
      MC<K> p2 = mul(a, load_aos<K>(x2, c));
      s1 = add(s1, p1);
      s2 = add(s2, p2);
      c = cn;
    }
  } else {
    // the two sums' lane chains one at a time (reference order, fewer live
    // accumulators), see lane4_row
    const int nfull = len >> 2;
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      MC<K> L1 = zero<K>(), L2 = zero<K>();
      for (int m = 0; m < nfull; ++m) {
        const int64_t e = (int64_t)(4 * m + j) * 16;
        MC<K> a = load_planes_stream<K>(vp, st, e);
        const int c = ld_s32_stream(cp + e);
        L1 = add(L1, mul(a, load_aos<K>(x1, c)));
        L2 = add(L2, mul(a, load_aos<K>(x2, c)));
      }
      s1 = add(s1, L1);
      s2 = add(s2, L2);
    }
    for (int k = nfull * 4; k < len; ++k) {
      const int64_t e = (int64_t)k * 16;
      MC<K> a = load_planes_stream<K>(vp, st, e);
      const int c = ld_s32_stream(cp + e);
      s1 = add(s1, mul(a, load_aos<K>(x1, c)));
      s2 = add(s2, mul(a, load_aos<K>(x2, c)));
    }
  }
  // re half: s1 = rr, s2 = ri; im half: s1 = ii, s2 = ir
  MC<K> o1 = shfl(s1, lane ^ 16);
  MC<K> o2 = shfl(s2, lane ^ 16);
  if (!imh && row >= 0) {
    store_aos<K>(yre, row, sub(s1, o1));  // rr - ii
    store_aos<K>(yim, row, add(s2, o2));  // ri + ir
  }
}

// ---------------------------------------------------------------------------
// Long rows, deterministic: one CTA per row.  All threads form the products
// of a chunk into shared memory (they are independent); the reference's
// serial add chains then run on 1 (SCALAR) or 4 (LANE4) threads per sum.
// ---------------------------------------------------------------------------
template <int K, bool CPLX>
MPSG_DI void long_products(const LongView& L, int64_t k, const double* __restrict__ xre,
                           const double* __restrict__ xim, MC<K>* out) {
  const int c = L.col[k];
  MC<K> are = load_planes<K>(L.val, L.stride, k);
  if constexpr (!CPLX) {
    out[0] = mul(are, load_aos<K>(xre, c));
  } else {
    MC<K> aim = load_planes<K>(L.val + (int64_t)K * L.stride, L.stride, k);
    MC<K> vr = load_aos<K>(xre, c), vi = load_aos<K>(xim, c);
    out[0] = mul(are, vr);  // rr
    out[1] = mul(aim, vi);  // ii
    out[2] = mul(are, vi);  // ri
    out[3] = mul(aim, vr);  // ir
  }
}

template <int K, int ORDER, bool CPLX, int CH>
__global__ void __launch_bounds__(128) long_det_kernel(LongView L, const double* __restrict__ xre,
                                                       const double* __restrict__ xim,
                                                       double* __restrict__ yre,
                                                       double* __restrict__ yim) {
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
  int64_t c0 = 0;
  for (; c0 < len; c0 += CH) {
    const int cnt = (int)((len - c0) < CH ? (len - c0) : CH);
    for (int i = tid; i < cnt; i += blockDim.x) long_products<K, CPLX>(L, b + c0 + i, xre, xim, prod + i * NS);
    __syncthreads();
    if (chain) {
      if constexpr (ORDER == ORDER_LANE4) {
        for (int i = lj; i < cnt && c0 + i < m4; i += 4) acc = add(acc, prod[i * NS + sidx]);
      } else {
        for (int i = 0; i < cnt; ++i) acc = add(acc, prod[i * NS + sidx]);
      }
    }
    if (c0 + CH < len) __syncthreads();
  }
  c0 -= CH;  // start of the last chunk (still resident in shared memory)
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
      if (tid == 0) {
        store_aos<K>(yre, L.row[r], sub(s, ii));
        store_aos<K>(yim, L.row[r], add(ri, ir));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Long rows, fast: one warp per chunk of L.chunk elements; lanes take strided
// elements (coalesced), a fixed xor-tree reduces the warp, and the last
// arriving warp of a row adds the chunk partials in chunk order.
// ---------------------------------------------------------------------------
#ifdef MPSG_LONG_MINB
#define MPSG_LONG_LB __launch_bounds__(128, MPSG_LONG_MINB)
#else
#define MPSG_LONG_LB __launch_bounds__(128)
#endif
template <int K, bool CPLX>
__global__ void MPSG_LONG_LB long_fast_kernel(LongView L, const double* __restrict__ xre,
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

  // U independent partial sums per lane (element k goes to partial
  // ((k - b) / 32) % U), so U gathers are in flight per thread; combined in
  // fixed order below.
#ifndef MPSG_LONG_U
#define MPSG_LONG_U 1
#endif
  constexpr int U = CPLX ? 1 : MPSG_LONG_U;
  MC<K> acc[NS];
  MC<K> pu[U][NS];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int s = 0; s < NS; ++s) pu[u][s] = zero<K>();
  int64_t k = b + lane;
  // column indices are loaded one round ahead (real case), so a round's
  // gathers issue as soon as it starts
  int cpf[U];
#pragma unroll
  for (int u = 0; u < U; ++u) cpf[u] = (!CPLX && k + 32 * u < e) ? ld_s32_stream(L.col + k + 32 * u) : 0;
  for (; k + 32 * (U - 1) < e; k += 32 * U) {
    int cnx[U];
    if constexpr (!CPLX) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t kn = k + 32 * (U + u);
        cnx[u] = kn < e ? ld_s32_stream(L.col + kn) : 0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t kk = k + 32 * u;
      MC<K> are = load_planes_stream<K>(L.val, L.stride, kk);
      if constexpr (!CPLX) {
        pu[u][0] = add(pu[u][0], mul(are, load_aos<K>(xre, cpf[u])));
      } else {
        const int c = ld_s32_stream(L.col + kk);
        MC<K> aim = load_planes_stream<K>(L.val + (int64_t)K * L.stride, L.stride, kk);
        MC<K> vr = load_aos<K>(xre, c), vi = load_aos<K>(xim, c);
        pu[u][0] = add(pu[u][0], mul(are, vr));
        pu[u][1] = add(pu[u][1], mul(aim, vi));
        pu[u][2] = add(pu[u][2], mul(are, vi));
        pu[u][3] = add(pu[u][3], mul(aim, vr));
      }
    }
    if constexpr (!CPLX) {
#pragma unroll
      for (int u = 0; u < U; ++u) cpf[u] = cnx[u];
    }
  }
#pragma unroll
  for (int u = 0; u < U - 1; ++u) {  // remainder: at most U-1 more elements per lane
    const int64_t kk = k + 32 * u;
    if (kk < e) {
      MC<K> are = load_planes_stream<K>(L.val, L.stride, kk);
      pu[u][0] = add(pu[u][0], mul(are, load_aos<K>(xre, cpf[u])));
    }
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    acc[s] = pu[0][s];
#pragma unroll
    for (int u = 1; u < U; ++u) acc[s] = add(acc[s], pu[u][s]);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = add(acc[s], shfl_xor(acc[s], off));

  auto finish = [&](MC<K>* sums) {
    const int row = L.row[r];
    if constexpr (!CPLX) {
      store_aos<K>(yre, row, sums[0]);
    } else {
      store_aos<K>(yre, row, sub(sums[0], sums[1]));
      store_aos<K>(yim, row, add(sums[2], sums[3]));
    }
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
