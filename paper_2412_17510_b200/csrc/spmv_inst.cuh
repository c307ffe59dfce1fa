// spmv_inst.cuh -- SpMV launch template, instantiated per K by spmv_k{2,3,4}.cu.
#pragma once
#include "internal.h"
#include "spmv_kernels.cuh"

#include <cstdlib>

#ifndef MPSG_FUSED
#define MPSG_FUSED 1
#endif

namespace mpsg {

// Launch every kernel of one SpMV over the device layout of A (layout.h):
// the long-row kernel on the context's aux stream (forked/joined by events)
// concurrently with the SELL kernel on `st`.  part = -2: all of it;
// part = -1: only the long-row kernel, on `st`; part >= 0: only the SELL
// slices of output part `part` (host-call overlap, capi.cu).
inline bool td_pad_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MPSG_TD_PAD");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <int K, bool CPLX, bool MX, bool CONJ>
int launch_spmv_mode(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* xre, const double* xim,
                     double* yre, double* yim, cudaStream_t st, int part) {
  const bool has_long = A->nlong > 0 && part < 0;
  const bool fork = has_long && part == -2;
  cudaStream_t lst = fork ? ctx->aux : st;
  // x (re, then im for complex: one window over the first, the hotter, is
  // all a launch can carry) -- see launch_win; off unless MPSG_L2_PERSIST=1
  const size_t xb = (size_t)A->ncols * K * sizeof(double);
  if (has_long) {
    if (fork) {
      CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, st));
      CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
    }
    LongView L = A->lng();
    if (order == ORDER_FAST) {
      const int blocks = (int)((A->nchunks + 3) / 4);
      CUDA_TRY(ctx, launch_win(ctx, long_fast_kernel<K, CPLX, MX, CONJ>, blocks, 128, 0, lst, xre, xb, L, xre, xim,
                               yre, yim));
    } else {
      constexpr int CH = CPLX ? 256 : 512;
      const size_t smem = (size_t)CH * (CPLX ? 4 : 1) * sizeof(MC<K>);
      if (order == ORDER_SCALAR && ctx->seg_T > 1)
        long_det_kernel<K, ORDER_SCALAR, CPLX, CH, MX, CONJ, true>
            <<<(int)A->nlong, MPSG_LONG_DET_THREADS, smem, lst>>>(L, xre, xim, yre, yim, ctx->seg_bounds, ctx->seg_T);
      else if (order == ORDER_SCALAR)
        long_det_kernel<K, ORDER_SCALAR, CPLX, CH, MX, CONJ>
            <<<(int)A->nlong, MPSG_LONG_DET_THREADS, smem, lst>>>(L, xre, xim, yre, yim);
      else
        long_det_kernel<K, ORDER_LANE4, CPLX, CH, MX, CONJ>
            <<<(int)A->nlong, MPSG_LONG_DET_THREADS, smem, lst>>>(L, xre, xim, yre, yim);
    }
    CUDA_TRY(ctx, cudaGetLastError());
    if (fork) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join, ctx->aux));
  }
  const SellView S = part >= 0 ? A->sell_range(A->part_slice[(size_t)part], A->part_slice[(size_t)part + 1])
                               : A->sell();
  // 256-bit x gathers (QD real kernels) need a 32-byte aligned x.  TD takes
  // them from the padded copy of x (mpsg_csr::xpad, FAST order, matrices with
  // enough gathers per column); a windowed 256-bit gather on the unpadded
  // [n][3] vector measured slower than three 64-bit loads.
  const bool xw = K == 4 && (reinterpret_cast<uintptr_t>(xre) & 31) == 0;
  if (part != -1 && S.nslices > 0) {
    const int blocks = (S.nslices + 3) / 4;
    // Short rows: ORDER_FAST walks them in the reference's lanes-off element
    // order (the faster of the two exact orders on B200 for every K,
    // profiles/r01b_variants.txt) but, with MPSG_FUSED=1 (the default), each
    // term goes through the fused product-accumulate fma_acc (mc_arith.cuh),
    // so the bits differ from lanes off and the result is held to the
    // componentwise bound instead; MPSG_FUSED=0 falls back to the exact
    // lanes-off chain.
    const int sorder = order == ORDER_FAST ? ORDER_SCALAR : order;
    const bool seg = order == ORDER_SCALAR && ctx->seg_T > 1;
    if constexpr (!CPLX) {
      if (seg)
        sell_real_seg_kernel<K, MX><<<blocks, 128, 0, st>>>(S, xre, yre, ctx->seg_bounds, ctx->seg_T);
      else if (order == ORDER_FAST && MPSG_FUSED && K == 3 && A->xpad && td_pad_enabled()) {
        if constexpr (K == 3) {
          // (host-call parts run in order on one stream: part 0 pads for all of them)
          if (part <= 0)
            pad_td_kernel<<<(unsigned)((A->ncols + 255) / 256), 256, 0, st>>>(xre, A->xpad, A->ncols);
          CUDA_TRY(ctx, launch_win(ctx, sell_real_kernel<K, ORDER_FAST, MX, true>, blocks, 128, 0, st, xre, xb, S,
                                   A->xpad, yre));
        }
      } else if (order == ORDER_FAST && MPSG_FUSED)
        CUDA_TRY(ctx, xw ? launch_win(ctx, sell_real_kernel<K, ORDER_FAST, MX, K == 4>, blocks, 128, 0, st, xre, xb, S,
                                      xre, yre)
                         : launch_win(ctx, sell_real_kernel<K, ORDER_FAST, MX, false>, blocks, 128, 0, st, xre, xb,
                                      S, xre, yre));
      else if (sorder == ORDER_SCALAR)
        CUDA_TRY(ctx, xw ? launch_win(ctx, sell_real_kernel<K, ORDER_SCALAR, MX, K == 4>, blocks, 128, 0, st, xre, xb,
                                      S, xre, yre)
                         : launch_win(ctx, sell_real_kernel<K, ORDER_SCALAR, MX, false>, blocks, 128, 0, st, xre, xb,
                                      S, xre, yre));
      else if constexpr (K == 2)
        CUDA_TRY(ctx, launch_win(ctx, sell_real_lane4_lat_kernel<K, MX>, blocks, 128, 0, st, xre, xb, S, xre, yre));
      else
        CUDA_TRY(ctx, xw ? launch_win(ctx, sell_real_kernel<K, ORDER_LANE4, MX, K == 4>, blocks, 128, 0, st, xre, xb,
                                      S, xre, yre)
                         : launch_win(ctx, sell_real_kernel<K, ORDER_LANE4, MX, false>, blocks, 128, 0, st, xre, xb,
                                      S, xre, yre));
    } else {
      if (seg)
        sell_complex_kernel<K, ORDER_SCALAR, MX, CONJ, true>
            <<<blocks, 128, 0, st>>>(S, xre, xim, yre, yim, ctx->seg_bounds, ctx->seg_T);
      else if (order == ORDER_FAST && MPSG_FUSED)
        CUDA_TRY(ctx, launch_win(ctx, sell_complex_kernel<K, ORDER_FAST, MX, CONJ>, blocks, 128, 0, st, xre, xb,
                                 S, xre, xim, yre, yim, nullptr, 1));
      else if (sorder == ORDER_SCALAR)
        CUDA_TRY(ctx, launch_win(ctx, sell_complex_kernel<K, ORDER_SCALAR, MX, CONJ>, blocks, 128, 0, st, xre, xb,
                                 S, xre, xim, yre, yim, nullptr, 1));
      else
        CUDA_TRY(ctx, launch_win(ctx, sell_complex_kernel<K, ORDER_LANE4, MX, CONJ>, blocks, 128, 0, st, xre, xb,
                                 S, xre, xim, yre, yim, nullptr, 1));
    }
    CUDA_TRY(ctx, cudaGetLastError());
  }
  if (fork) CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_join, 0));
  return MPSG_OK;
}

template <int K, bool CPLX>
int launch_spmv_k(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* xre, const double* xim,
                  double* yre, double* yim, cudaStream_t st, bool conj, int part) {
  if constexpr (CPLX) {
    if (A->mixed)
      return conj ? launch_spmv_mode<K, true, true, true>(ctx, A, order, xre, xim, yre, yim, st, part)
                  : launch_spmv_mode<K, true, true, false>(ctx, A, order, xre, xim, yre, yim, st, part);
    return conj ? launch_spmv_mode<K, true, false, true>(ctx, A, order, xre, xim, yre, yim, st, part)
                : launch_spmv_mode<K, true, false, false>(ctx, A, order, xre, xim, yre, yim, st, part);
  } else {
    if (A->mixed) return launch_spmv_mode<K, false, true, false>(ctx, A, order, xre, xim, yre, yim, st, part);
    return launch_spmv_mode<K, false, false, false>(ctx, A, order, xre, xim, yre, yim, st, part);
  }
}

}  // namespace mpsg

#define MPSG_INSTANTIATE_SPMV(K)                                                                            \
  template int mpsg::launch_spmv_k<K, false>(mpsg_ctx*, const mpsg_csr*, int, const double*, const double*, \
                                             double*, double*, cudaStream_t, bool, int);                     \
  template int mpsg::launch_spmv_k<K, true>(mpsg_ctx*, const mpsg_csr*, int, const double*, const double*,  \
                                            double*, double*, cudaStream_t, bool, int);
