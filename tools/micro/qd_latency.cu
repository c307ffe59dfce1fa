// Single-thread latency of the multi-component ops (development probe):
// cycles per dependent add / mul / divide / sqrt at K = 2, 4, and the cost
// of a fence + atomic ticket, to size the serial tail of the solver reductions.
#include <cstdio>
#include "../../paper_2412_17510_b200/csrc/mc_arith.cuh"
using namespace mpsg;

template <int K, int OP>
__global__ void chain(double* out, int n, long long* cyc) {
  MC<K> a, b;
  for (int j = 0; j < K; ++j) { a.c[j] = 1.0 + j * 1e-17; b.c[j] = 0.999 + j * 1e-18; }
  a.c[0] = out[0] + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) a = add(a, b);
    else if (OP == 1) a = mul(a, b);
    else if (OP == 2) a = divide(a, b);
    else if (OP == 3) a = sqrt_mc(a);
    else { __threadfence(); atomicAdd((unsigned*)out + 2, 1u); a.c[0] += 1.0; }
  }
  long long t1 = clock64();
  for (int j = 0; j < K; ++j) out[1] += a.c[j];
  *cyc = t1 - t0;
}

template <int K>
void run() {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 64); cudaMemset(d, 0, 64); cudaMalloc(&c, 8);
  const char* names[] = {"add", "mul", "divide", "sqrt", "fence+atomic"};
  for (int op = 0; op < 5; ++op) {
    const int n = 200;
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<K, 0><<<1, 1>>>(d, n, c); break;
        case 1: chain<K, 1><<<1, 1>>>(d, n, c); break;
        case 2: chain<K, 2><<<1, 1>>>(d, n, c); break;
        case 3: chain<K, 3><<<1, 1>>>(d, n, c); break;
        case 4: chain<K, 4><<<1, 1>>>(d, n, c); break;
      }
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    }
    printf("K=%d %-13s %8.1f cycles per op (dependent, one thread)\n", K, names[op], (double)h / n);
  }
}

int main() {
  run<2>();
  run<4>();
  return 0;
}
