// tools.cu -- measurement and verification entry points of the C ABI.
//
//  * mpsg_measure_fp64_peak: the fp64-pipe roofline denominator.  The driver's
//    MEASURED_PEAKS.json carries HBM and bf16 only, and TD/QD SpMV are
//    fp64-bound, so the peak is measured here on the box:
//    a grid of 16 blocks per SM, each thread running 8 independent DFMA
//    chains (latency hidden by ILP x occupancy), timed with CUDA events.
//    One DFMA counts as one fp64 operation, the unit the algorithmic op counts
//    use (20 / 202 / 206 ops per nonzero).
//  * mpsg_mc_op_dev: batched device MC arithmetic (add, mul, mul_by_double,
//    sub, divide, sqrt) so tests can pin every op bit-for-bit against the
//    reference, like the reference's lane-vs-scalar acceptance check 3.
#include <cuda_runtime.h>

#include "internal.h"
#include "mc_arith.cuh"

using namespace mpsg;

namespace {

__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999999, c = 1e-9;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    a0 = __fma_rn(a0, b, c);
    a1 = __fma_rn(a1, b, c);
    a2 = __fma_rn(a2, b, c);
    a3 = __fma_rn(a3, b, c);
    a4 = __fma_rn(a4, b, c);
    a5 = __fma_rn(a5, b, c);
    a6 = __fma_rn(a6, b, c);
    a7 = __fma_rn(a7, b, c);
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains live
}

template <int K>
__global__ void mc_op_kernel(int op, int64_t n, const double* a, const double* b, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  MC<K> x = load_aos_rw<K>(a, i), y = load_aos_rw<K>(b, i), r;
  switch (op) {
    case 0: r = add(x, y); break;
    case 1: r = mul(x, y); break;
    case 2: r = mul_d(x, y.c[0]); break;
    case 3: r = sub(x, y); break;
    case 4: r = divide(x, y); break;
    default: r = sqrt_mc(x); break;
  }
  store_aos<K>(out, i, r);
}

// The reference harness's input vectors (bench.hpp:78-111), evaluated with
// the device restatement of the reference ops, so the bits are the
// reference's: v_j = sqrt(2) * j; complex v_j = sqrt(2 + 3i) * j with
// Re = sqrt((sqrt(13) + 2) / 2), Im = sqrt((sqrt(13) - 2) / 2).
template <int K>
__global__ void make_vector_kernel(int64_t n, double* re, double* im) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const MC<K> j = from_double<K>((double)(i + 1));
  if (!im) {
    store_aos<K>(re, i, mul(sqrt_mc(from_double<K>(2.0)), j));
    return;
  }
  const MC<K> half = from_double<K>(0.5), two = from_double<K>(2.0);
  const MC<K> root13 = sqrt_mc(from_double<K>(13.0));
  const MC<K> r = sqrt_mc(mul(add(root13, two), half));
  const MC<K> m = sqrt_mc(mul(sub(root13, two), half));
  store_aos<K>(re, i, mul(r, j));
  store_aos<K>(im, i, mul(m, j));
}

}  // namespace

extern "C" {

MPSG_API int mpsg_make_vector(mpsg_ctx* ctx, int K, int64_t n, double* re, double* im) {
  if (!ctx || !re || n < 1) return MPSG_E_ARG;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  const size_t b = (size_t)n * K * sizeof(double);
  double *d = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&d, b * (im ? 2 : 1)));
  cudaStream_t st = ctx->stream;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  double* dim = im ? d + (size_t)n * K : nullptr;
  switch (K) {
    case 2: make_vector_kernel<2><<<blocks, 128, 0, st>>>(n, d, dim); break;
    case 3: make_vector_kernel<3><<<blocks, 128, 0, st>>>(n, d, dim); break;
    case 4: make_vector_kernel<4><<<blocks, 128, 0, st>>>(n, d, dim); break;
    default: cudaFree(d); return fail(ctx, MPSG_E_ARG, "make_vector: K must be 2, 3 or 4");
  }
  cudaError_t e = cudaMemcpyAsync(re, d, b, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && im) e = cudaMemcpyAsync(im, dim, b, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d);
  if (e != cudaSuccess) return fail(ctx, MPSG_E_CUDA, "make_vector: %s", cudaGetErrorString(e));
  return MPSG_OK;
}

MPSG_API int mpsg_measure_fp64_peak(mpsg_ctx* ctx, double* ops_per_s) {
  if (!ctx || !ops_per_s) return MPSG_E_ARG;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  int sms = 0;
  CUDA_TRY(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const int blocks = sms * 16, threads = 256, iters = 4096;
  double* out = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&out, blocks * sizeof(double)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStream_t st = ctx->stream;
  fp64_peak_kernel<<<blocks, threads, 0, st>>>(out, iters, 1.0);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, st);
    fp64_peak_kernel<<<blocks, threads, 0, st>>>(out, iters, 1.0 + rep);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) return fail(ctx, MPSG_E_CUDA, "fp64 peak: %s", cudaGetErrorString(e));
  *ops_per_s = (double)blocks * threads * iters * 8.0 / (best * 1e-3);
  return MPSG_OK;
}

// Batched device MC ops on AoS device arrays: op 0 add, 1 mul, 2 mul_by_double
// (b's leading component), 3 sub, 4 divide, 5 sqrt(a).
MPSG_API int mpsg_mc_op_dev(mpsg_ctx* ctx, int op, int K, int64_t n, const double* d_a,
                            const double* d_b, double* d_out) {
  if (!ctx || op < 0 || op > 5) return MPSG_E_ARG;
  if (n == 0) return MPSG_OK;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  cudaStream_t st = ctx->stream;
  switch (K) {
    case 2: mc_op_kernel<2><<<blocks, 128, 0, st>>>(op, n, d_a, d_b, d_out); break;
    case 3: mc_op_kernel<3><<<blocks, 128, 0, st>>>(op, n, d_a, d_b, d_out); break;
    case 4: mc_op_kernel<4><<<blocks, 128, 0, st>>>(op, n, d_a, d_b, d_out); break;
    default: return fail(ctx, MPSG_E_ARG, "mc_op: K must be 2, 3 or 4");
  }
  CUDA_TRY(ctx, cudaGetLastError());
  return MPSG_OK;
}

}  // extern "C"
