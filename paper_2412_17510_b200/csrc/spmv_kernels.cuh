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
  for (int j = 0; j < K; ++j) a.c[j] = __ldcs(val + j * stride + e);
  return a;
}

// ---------------------------------------------------------------------------
// SELL slice, real: one warp per slice of 32 rows, one thread per row.
// ---------------------------------------------------------------------------
template <int K, int ORDER>
__global__ void __launch_bounds__(128) sell_real_kernel(SellView S, const double* __restrict__ x,
                                                        double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= S.nslices) return;
  const int slot = s * 32 + lane;
  const int row = S.slot_row[slot];
  const int len = S.slot_len[slot];
  const int64_t base = S.slice_ptr[s] + lane;
  const int* __restrict__ cp = S.col + base;
  const double* __restrict__ vp = S.val + base;
  const int64_t st = S.stride;

  MC<K> acc = zero<K>();
  if constexpr (ORDER == ORDER_SCALAR) {
    int k = 0;
    for (; k + 4 <= len; k += 4) {
      MC<K> p[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t e = (int64_t)(k + j) * 32;
        MC<K> a = load_planes_stream<K>(vp, st, e);
        MC<K> xv = load_aos<K>(x, __ldcs(cp + e));
        p[j] = mul(a, xv);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) acc = add(acc, p[j]);
    }
    for (; k < len; ++k) {
      const int64_t e = (int64_t)k * 32;
      MC<K> a = load_planes_stream<K>(vp, st, e);
      MC<K> xv = load_aos<K>(x, __ldcs(cp + e));
      acc = add(acc, mul(a, xv));
    }
  } else {
    MC<K> L[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) L[j] = zero<K>();
    const int m4 = len & ~3;
    for (int k = 0; k < m4; k += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t e = (int64_t)(k + j) * 32;
        MC<K> a = load_planes_stream<K>(vp, st, e);
        MC<K> xv = load_aos<K>(x, __ldcs(cp + e));
        L[j] = add(L[j], mul(a, xv));
      }
    }
    acc = add(add(add(add(acc, L[0]), L[1]), L[2]), L[3]);
    for (int k = m4; k < len; ++k) {
      const int64_t e = (int64_t)k * 32;
      MC<K> a = load_planes_stream<K>(vp, st, e);
      MC<K> xv = load_aos<K>(x, __ldcs(cp + e));
      acc = add(acc, mul(a, xv));
    }
  }
  if (row >= 0) store_aos<K>(y, row, acc);
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
    for (int k = 0; k < len; ++k) {
      const int64_t e = (int64_t)k * 16;
      MC<K> a = load_planes_stream<K>(vp, st, e);
      const int c = __ldcs(cp + e);
      MC<K> p1 = mul(a, load_aos<K>(x1, c));
      MC<K> p2 = mul(a, load_aos<K>(x2, c));
      s1 = add(s1, p1);
      s2 = add(s2, p2);
    }
  } else {
    MC<K> L1[4], L2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) L1[j] = L2[j] = zero<K>();
    const int m4 = len & ~3;
    for (int k = 0; k < m4; k += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t e = (int64_t)(k + j) * 16;
        MC<K> a = load_planes_stream<K>(vp, st, e);
        const int c = __ldcs(cp + e);
        L1[j] = add(L1[j], mul(a, load_aos<K>(x1, c)));
        L2[j] = add(L2[j], mul(a, load_aos<K>(x2, c)));
      }
    }
    s1 = add(add(add(add(s1, L1[0]), L1[1]), L1[2]), L1[3]);
    s2 = add(add(add(add(s2, L2[0]), L2[1]), L2[2]), L2[3]);
    for (int k = m4; k < len; ++k) {
      const int64_t e = (int64_t)k * 16;
      MC<K> a = load_planes_stream<K>(vp, st, e);
      const int c = __ldcs(cp + e);
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
template <int K, bool CPLX>
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
  const int64_t rb = L.ptr[r], re = L.ptr[r + 1];
  const int64_t b = rb + (int64_t)(w - first) * L.chunk;
  const int64_t e = (b + L.chunk < re) ? b + L.chunk : re;

  MC<K> acc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) acc[s] = zero<K>();
  for (int64_t k = b + lane; k < e; k += 32) {
    const int c = __ldcs(L.col + k);
    MC<K> are = load_planes_stream<K>(L.val, L.stride, k);
    if constexpr (!CPLX) {
      acc[0] = add(acc[0], mul(are, load_aos<K>(xre, c)));
    } else {
      MC<K> aim = load_planes_stream<K>(L.val + (int64_t)K * L.stride, L.stride, k);
      MC<K> vr = load_aos<K>(xre, c), vi = load_aos<K>(xim, c);
      acc[0] = add(acc[0], mul(are, vr));
      acc[1] = add(acc[1], mul(aim, vi));
      acc[2] = add(acc[2], mul(are, vi));
      acc[3] = add(acc[3], mul(aim, vr));
    }
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
  double* part = L.partial + (int64_t)w * NS * K;
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
