// spmv_inst.cuh -- SpMV launch template, instantiated per K by spmv_k{2,3,4}.cu.
#pragma once
#include "internal.h"
#include "spmv_kernels.cuh"

namespace mpsg {

template <int K, bool CPLX>
int launch_spmv_k(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* xre,
                  const double* xim, double* yre, double* yim, cudaStream_t st) {
  const bool has_long = A->nlong > 0;
  if (has_long) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, st));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
    LongView L = A->lng();
    if (order == ORDER_FAST) {
      const int blocks = (int)((A->nchunks + 3) / 4);
      long_fast_kernel<K, CPLX><<<blocks, 128, 0, ctx->aux>>>(L, xre, xim, yre, yim);
    } else {
      constexpr int CH = CPLX ? 256 : 512;
      const size_t smem = (size_t)CH * (CPLX ? 4 : 1) * sizeof(MC<K>);
      if (order == ORDER_SCALAR)
        long_det_kernel<K, ORDER_SCALAR, CPLX, CH><<<(int)A->nlong, 128, smem, ctx->aux>>>(L, xre, xim, yre, yim);
      else
        long_det_kernel<K, ORDER_LANE4, CPLX, CH><<<(int)A->nlong, 128, smem, ctx->aux>>>(L, xre, xim, yre, yim);
    }
    CUDA_TRY(ctx, cudaGetLastError());
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join, ctx->aux));
  }
  if (A->nslices > 0) {
    const int blocks = (int)((A->nslices + 3) / 4);
    SellView S = A->sell();
    if constexpr (!CPLX) {
      if (order == ORDER_SCALAR)
        sell_real_kernel<K, ORDER_SCALAR><<<blocks, 128, 0, st>>>(S, xre, yre);
      else
        sell_real_kernel<K, ORDER_LANE4><<<blocks, 128, 0, st>>>(S, xre, yre);
    } else {
      if (order == ORDER_SCALAR)
        sell_complex_kernel<K, ORDER_SCALAR><<<blocks, 128, 0, st>>>(S, xre, xim, yre, yim);
      else
        sell_complex_kernel<K, ORDER_LANE4><<<blocks, 128, 0, st>>>(S, xre, xim, yre, yim);
    }
    CUDA_TRY(ctx, cudaGetLastError());
  }
  if (has_long) CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_join, 0));
  return MPSG_OK;
}


}  // namespace mpsg

#define MPSG_INSTANTIATE_SPMV(K)                                                              \
  template int mpsg::launch_spmv_k<K, false>(mpsg_ctx*, const mpsg_csr*, int, const double*,   \
                                             const double*, double*, double*, cudaStream_t);   \
  template int mpsg::launch_spmv_k<K, true>(mpsg_ctx*, const mpsg_csr*, int, const double*,    \
                                            const double*, double*, double*, cudaStream_t);
