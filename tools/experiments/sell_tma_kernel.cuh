// EXPERIMENT (not built into libmpsg.so): FAST short rows with the matrix
// stream staged through shared memory by bulk copies, one ring per warp.
// Measured on B200 (profiles/r02_variants.txt, items 15-16): cfg2 QD 303 us
// against the plain kernel's 293 us, TD 226 against 196.  It needs
// csrc/async_copy.cuh (next to this file) and the launcher removed from
// spmv_inst.cuh in the same commit.
// ---------------------------------------------------------------------------
// FAST short rows with the matrix stream staged through shared memory by bulk
// copies (TMA), TD/QD.  In sell_real_kernel every product's operands are
// requested right before use (the 64-register cap leaves no room to hold the
// next product's), so a warp waits a full HBM round trip per product.  The
// value planes are 80% of the bytes and perfectly predictable: each warp keeps
// a ring of S stages of G rounds (one round = element k of its 32 rows, 256
// bytes per plane, contiguous in the SELL layout) filled by one elected lane
// with one bulk copy per plane per stage, S stages ahead, completion on the
// stage's mbarrier -- no registers are held across the HBM latency and the
// loop reads a from shared memory (K conflict-free LDS.64).  Only the x
// gathers (L2-resident for the benchmark sizes) and the column indices (a
// round group ahead, as before) still come through registers.  The warp walks
// the slice's width together; lanes past their row's end skip the arithmetic.
// ---------------------------------------------------------------------------
#ifndef MPSG_TMA_G
#define MPSG_TMA_G 2
#endif
#ifndef MPSG_TMA_S
#define MPSG_TMA_S 2
#endif
#ifndef MPSG_TMA_MINB
#define MPSG_TMA_MINB 8
#endif
template <int K, bool MX>
constexpr int sell_tma_smem_bytes() {
  return 4 * MPSG_TMA_S * MPSG_TMA_G * (MX ? 1 : K) * 256 + 4 * MPSG_TMA_S * 8;
}
template <int K, bool MX, bool XW>
__global__ void __launch_bounds__(128, MPSG_TMA_MINB)
    sell_real_tma_kernel(SellView Sv, const double* __restrict__ x, double* __restrict__ y) {
  constexpr int G = MPSG_TMA_G, S = MPSG_TMA_S;
  constexpr int NPL = MX ? 1 : K;
  constexpr int STGB = G * NPL * 256;  // bytes per stage: [plane][round][lane]
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wsm = smem + warp * S * STGB;
  const uint32_t wsm32 = ac::smem_u32(wsm);
  const uint32_t bar0 = ac::smem_u32(smem) + 4 * S * STGB + warp * S * 8;  // this warp's full[S]
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < S; ++i) ac::mbar_init(bar0 + i * 8, 1);
    ac::fence_mbar_init();
  }
  __syncwarp();
  const int s = blockIdx.x * 4 + warp;
  if (s >= Sv.nslices) return;
  const int64_t base = Sv.slice_ptr[s];
  const int w = (int)((Sv.slice_ptr[s + 1] - base) >> 5);  // slice width in rounds
  const int ngroups = (w + G - 1) / G;
  const int slot = s * 32 + lane;
  const int row = Sv.slot_row[slot];
  const int len = Sv.slot_len[slot];
  const int* __restrict__ cp = Sv.col + base + lane;
  auto issue = [&](int g) {  // rounds [g*G, min((g+1)*G, w)) of every plane into stage g % S
    if (g < ngroups && ac::elect_one()) {
      const int rounds = min(G, w - g * G);
      const uint32_t bar = bar0 + (g % S) * 8, dst = wsm32 + (g % S) * STGB;
      ac::mbar_arrive_expect_tx(bar, (uint32_t)(rounds * NPL * 256));
#pragma unroll
      for (int j = 0; j < NPL; ++j)
        ac::bulk_g2s(dst + j * (G * 256), Sv.val + (int64_t)j * Sv.stride + base + (int64_t)g * (G * 32),
                     (uint32_t)(rounds * 256), bar);
    }
  };
#pragma unroll
  for (int g = 0; g < S; ++g) issue(g);
  int c[G];
#pragma unroll
  for (int j = 0; j < G; ++j) c[j] = j < w ? ld_s32_stream(cp + (int64_t)j * 32) : 0;
  MC<K> acc = zero<K>();
  for (int g = 0; g < ngroups; ++g) {
    int cn[G];
#pragma unroll
    for (int j = 0; j < G; ++j) cn[j] = ((g + 1) * G + j < w) ? ld_s32_stream(cp + (int64_t)((g + 1) * G + j) * 32) : 0;
    MC<K> v[G];
#pragma unroll
    for (int j = 0; j < G; ++j) v[j] = load_x<K>(x, XW, c[j]);  // padding rounds gather x[0]
    ac::mbar_wait(bar0 + (g % S) * 8, (uint32_t)(g / S) & 1u);
    const unsigned char* stg = wsm + (g % S) * STGB;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      AVal<K, MX> a;
      if constexpr (MX) {
        a.a = reinterpret_cast<const double*>(stg + j * 256)[lane];
      } else {
#pragma unroll
        for (int q = 0; q < K; ++q) a.a.c[q] = reinterpret_cast<const double*>(stg + (q * G + j) * 256)[lane];
      }
      if (g * G + j < len) a.accumulate_lvl(acc, v[j]);
    }
    if (G >= 4 || (g & 1)) acc = lvl_sweep(acc);
    __syncwarp();
    ac::fence_proxy_async();
    issue(g + S);
#pragma unroll
    for (int j = 0; j < G; ++j) c[j] = cn[j];
  }
  acc = canon(lvl_sweep(acc));
  if (row >= 0) store_aos<K>(y, row, acc);
}

