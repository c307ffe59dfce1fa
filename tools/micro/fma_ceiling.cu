// fp64-pipe ceiling of the FAST QD/TD accumulate without memory (development
// probe): every thread runs the same serial chain of fma_acc as the SELL
// kernel (G products per round, operands rotated in registers), at a chosen
// number of resident warps; prints fp64 instructions per second and the
// fraction of the DFMA peak measured the same way.  Tells whether the QD
// kernel's 76% fp64-pipe activity is a memory limit or an issue limit.
#include <cstdio>
#include "../../paper_2412_17510_b200/csrc/mc_arith.cuh"
using namespace mpsg;

template <int K, int G, int MINB>
__global__ void __launch_bounds__(128, MINB) chain(double* out, int n) {
  MC<K> a[G], x[G];
  const double t = threadIdx.x * 1e-3 + blockIdx.x * 1e-6;
  for (int g = 0; g < G; ++g)
    for (int j = 0; j < K; ++j) {
      a[g].c[j] = (1.0 + g + t) * ldexp(1.0, -53 * j);
      x[g].c[j] = (0.7 - g * 0.1 + t) * ldexp(1.0, -53 * j);
    }
  MC<K> acc = zero<K>();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int g = 0; g < G; ++g) acc = fma_acc(acc, a[g], x[g]);
    // rotate one operand so the compiler cannot hoist anything
    MC<K> tmp = a[0];
#pragma unroll
    for (int g = 0; g + 1 < G; ++g) a[g] = a[g + 1];
    a[G - 1] = tmp;
  }
  double s = 0;
  for (int j = 0; j < K; ++j) s += acc.c[j];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_peak(double* out, int n) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < n; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1.2345) out[0] = 1;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

template <int K, int G, int MINB>
void run(double peak, int ops_per_acc, int sms) {
  double* d;
  cudaMalloc(&d, 64);
  const int n = 2000, blocks = sms * MINB;
  float ms = timeit([&] { chain<K, G, MINB><<<blocks, 128>>>(d, n); });
  const double ops = (double)blocks * 128 * n * G * ops_per_acc;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, chain<K, G, MINB>);
  printf("K=%d G=%d blocks/SM=%2d regs=%3d local=%3zu: %.2f T fp64 ops/s = %.3f of the DFMA peak\n", K, G, MINB,
         fa.numRegs, fa.localSizeBytes, ops / ms / 1e9, ops / ms / 1e9 / peak);
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  const int n = 20000, blocks = sms * 8;
  float ms = timeit([&] { dfma_peak<<<blocks, 256>>>(d, n); });
  const double peak = (double)blocks * 256 * n * 8 / ms / 1e9;
  printf("DFMA peak %.2f T/s (%d SMs)\n", peak, sms);
  run<4, 4, 8>(peak, 121, sms);
  run<4, 4, 4>(peak, 121, sms);
  run<4, 4, 2>(peak, 121, sms);
  run<4, 4, 1>(peak, 121, sms);
  run<4, 2, 8>(peak, 121, sms);
  run<4, 1, 8>(peak, 121, sms);
  run<4, 1, 12>(peak, 121, sms);
  run<3, 2, 8>(peak, 52, sms);
  run<3, 2, 4>(peak, 52, sms);
  return 0;
}
