// spmv_ws.cuh -- warp-specialised FAST-order SELL kernel (real, short rows).
//
// The plain FAST kernel (sell_real_kernel<K, ORDER_FAST>) is latency-limited
// for TD/QD: under its 64-register cap a thread cannot hold the next
// products' operands while it runs the current 121-operation accumulate, so
// every product pays a full HBM round trip (ncu r01l: 8.7 of 16.5 stall
// cycles per instruction on the long scoreboard, fp64 pipe 75% busy).  Here
// the loads leave the arithmetic warps altogether:
//
//  * a CTA is NC consumer warps (one SELL slice of 32 rows each, one thread
//    per row, the lanes-off element order) + 1 producer warp;
//  * per consumer a ring of S stages in shared memory, one product round
//    (element k of all 32 rows) per stage: the slice's value planes arrive by
//    one 256-byte bulk copy per plane (cp.async.bulk, elected lane, mbarrier
//    complete_tx -- the SELL layout makes each per-k plane segment
//    contiguous), the gathered x[col] by per-lane cp.async straight into
//    shared memory (no registers held across the HBM latency), tracked by the
//    same mbarrier (cp.async.mbarrier.arrive.noinc);
//  * the producer prefetches the column indices S rounds ahead in registers
//    (coalesced 128-byte loads) -- the consumers never see them;
//  * consumers wait on the stage's `full` barrier, read a (K conflict-free
//    LDS.64) and x (LDS.128 halves / LDS.64 for TD), run the level-wise
//    accumulate, and release the stage (`empty` barrier, one arrive per warp).
//
// Arithmetic: fma_lvl (mc_arith.cuh) -- the level sums of fma_acc kept
// unnormalised across a group of S products, one backward sweep per group,
// canon() once per row.
#pragma once

#include "layout.h"
#include "mc_arith.cuh"

namespace mpsg {
namespace ws {

MPSG_DI uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
MPSG_DI void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
MPSG_DI void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
MPSG_DI void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}
MPSG_DI void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared, completion counted in bytes on `bar`
MPSG_DI void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
MPSG_DI void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
MPSG_DI void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
// the executing thread's earlier cp.asyncs arrive on `bar` when they land
// (.noinc: the arrival was counted in the barrier's initial count)
MPSG_DI void cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
MPSG_DI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
MPSG_DI void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// one elected lane of the (converged) warp: lets the compiler issue the bulk
// copies from uniform registers without a per-lane loop
MPSG_DI bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

template <int K>
struct XPieces {  // how one x element (K doubles) is cut into cp.async pieces
  static constexpr int PB = (K % 2 == 0) ? 16 : 8;  // piece bytes
  static constexpr int NP = K * 8 / PB;             // pieces per element
};

// cp.async groups (items) the producer keeps in flight
// (0: no groups -- each lane's gathers arrive on the stage's barrier by
// themselves, cp.async.mbarrier.arrive.noinc, so an item becomes visible
// without the producer having to come back to it)
#ifndef MPSG_WS_D
#define MPSG_WS_D 0
#endif
#ifndef MPSG_WS_MINB
#define MPSG_WS_MINB 0
#endif

// Shared memory per CTA: NC * S stages of (NPL + K) * 256 bytes, the column
// ring (NC consumers x 2 blocks x S rounds x 128 bytes), then the barriers
// (full[NC][S], empty[NC][S], colbar[NC][2]).
template <int K, bool MX, int NC, int S>
constexpr int ws_smem_bytes() {  // (independent of the number of producer warps)
  return NC * S * ((MX ? 1 : K) + K) * 256 + NC * 2 * S * 128 + (2 * NC * S + 2 * NC) * 8;
}

// x gathers in flight per producer warp (register sets of K doubles)
#ifndef MPSG_WS_P
#define MPSG_WS_P 4
#endif

// XPAD: x elements are 32 bytes apart (QD, or the padded TD copy) and are
// gathered with one 256-bit load; otherwise K 64-bit loads (TD, [n][3]).
template <int K, bool MX, int NC, int S, int NPW, bool XPAD>
__global__ void __launch_bounds__((NC + NPW) * 32, MPSG_WS_MINB)
    sell_ws_kernel(SellView Sv, const double* __restrict__ x, double* __restrict__ y) {
  constexpr int NPL = MX ? 1 : K;
  constexpr int A_BYTES = NPL * 256;
  constexpr int STG = A_BYTES + K * 256;
  constexpr int PB = XPieces<K>::PB, NP = XPieces<K>::NP;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t colb0 = sbase + NC * S * STG;      // column block (c, buf) at colb0 + (c*2+buf)*S*128
  const uint32_t bar0 = colb0 + NC * 2 * S * 128;   // full[c][i] at bar0 + (c*S+i)*8, empty after them
  const uint32_t cbar0 = bar0 + 2 * NC * S * 8;     // colbar[c][buf]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NC * S; ++i) {
      mbar_init(bar0 + i * 8, 33);               // 32 producer-lane arrivals + the elected lane's expect_tx
      mbar_init(bar0 + (NC * S + i) * 8, 1);     // the consumer warp's release
    }
    for (int i = 0; i < NC * 2; ++i) mbar_init(cbar0 + i * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int s0 = blockIdx.x * NC;
  const int ncons = min(NC, Sv.nslices - s0);  // live consumers (the last CTA may have fewer)

  if (warp >= NC) {
    // ------------------------------ producer ------------------------------
    // NPW producer warps, each serving NCP = NC / NPW consecutive consumers.
    // Items (round r, consumer c) are visited in the fixed order r*NCP + c
    // (items past a slice's width are empty).  Visiting item t: (1) the item
    // P places back is retired -- its gathered x, held in registers since,
    // goes to its stage and every lane arrives on the stage's `full` barrier;
    // (2) item t is issued: wait for its stage (`empty`), one elected lane
    // starts the bulk copies of the value planes (complete_tx on `full`), and
    // every lane starts its x gather (one 256-bit load = one L1 wavefront per
    // element; cp.async straight to shared memory can only move 16 bytes per
    // instruction -- two wavefronts per QD element, three per TD element --
    // and measured L1-bound on random columns: cfg2 QD 340 us).  P gathers
    // stay in flight per lane.  The column indices reach the producer through
    // shared memory (one bulk copy per S rounds, two blocks per consumer, a
    // block ahead).
    static_assert(NC % NPW == 0, "consumers must divide among the producer warps");
    constexpr int NCP = NC / NPW;
    const int cb = (warp - NC) * NCP;  // first consumer served
    constexpr int NI = NCP * S;        // items per unrolled pass
    constexpr int P = MPSG_WS_P;
    static_assert(NI % P == 0 && P < NI, "register sets must map statically onto the items of a pass");
    int64_t base[NCP];
    int w[NCP];
    int maxw = 0;
#pragma unroll
    for (int c = 0; c < NCP; ++c) {
      if (cb + c < ncons) {
        base[c] = Sv.slice_ptr[s0 + cb + c];
        w[c] = (int)((Sv.slice_ptr[s0 + cb + c + 1] - base[c]) >> 5);
      } else {
        base[c] = 0;
        w[c] = 0;
      }
      maxw = max(maxw, w[c]);
    }
    // column block b of consumer c: rounds [b*S, min((b+1)*S, w[c]))
    auto issue_cols = [&](int c, int b) {
      if (b * S < w[c] && elect_one()) {
        const uint32_t bytes = (uint32_t)min(S, w[c] - b * S) * 128u;
        const uint32_t bar = cbar0 + ((cb + c) * 2 + (b & 1)) * 8;
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s(colb0 + ((cb + c) * 2 + (b & 1)) * (S * 128), Sv.col + base[c] + (int64_t)b * (S * 32), bytes, bar);
      }
    };
#pragma unroll
    for (int c = 0; c < NCP; ++c) {
      issue_cols(c, 0);
      issue_cols(c, 1);
    }
    MC<K> xr[P];
    auto retire = [&](int mc, int mi, const MC<K>& v) {
      const uint32_t stg = sbase + ((cb + mc) * S + mi) * STG + A_BYTES;
      if constexpr (PB == 16) {
#pragma unroll
        for (int p = 0; p < NP; ++p)
          asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(stg + p * 512 + lane * 16), "d"(v.c[2 * p]),
                       "d"(v.c[2 * p + 1])
                       : "memory");
      } else {
#pragma unroll
        for (int p = 0; p < NP; ++p)
          asm volatile("st.shared.f64 [%0], %1;" ::"r"(stg + p * 256 + lane * 8), "d"(v.c[p]) : "memory");
      }
      mbar_arrive(bar0 + ((cb + mc) * S + mi) * 8);
    };
    for (int r0 = 0; r0 < maxw; r0 += S) {
      const int b = r0 / S;
      const uint32_t ph = (uint32_t)b & 1u;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const int r = r0 + i;
#pragma unroll
        for (int c = 0; c < NCP; ++c) {
          const int t = i * NCP + c;
          {  // (1) retire the item P places back
            const int m = (t - P + NI) % NI;
            const int mc = m % NCP, mi = m / NCP;
            const int mr = (t >= P) ? r0 + mi : r0 - S + mi;  // its round
            if (mr >= 0 && mr < w[mc]) retire(mc, mi, xr[t % P]);
          }
          if (r < w[c]) {  // (2) issue
            const uint32_t full = bar0 + ((cb + c) * S + i) * 8, empty = full + NC * S * 8;
            const uint32_t stg = sbase + ((cb + c) * S + i) * STG;
            if (i == 0) mbar_wait(cbar0 + ((cb + c) * 2 + (b & 1)) * 8, (uint32_t)(b >> 1) & 1u);
            const int col = *reinterpret_cast<const int*>(smem + NC * S * STG +
                                                          (((cb + c) * 2 + (b & 1)) * S + i) * 128 + lane * 4);
            mbar_wait(empty, ph ^ 1u);
            if (elect_one()) {
              mbar_arrive_expect_tx(full, A_BYTES);
#pragma unroll
              for (int j = 0; j < NPL; ++j)
                bulk_g2s(stg + j * 256, Sv.val + (int64_t)j * Sv.stride + base[c] + 32 * r, 256, full);
            }
            if constexpr (XPAD)
              xr[t % P] = load_x_wide<K>(x, col);
            else
              xr[t % P] = load_aos<K>(x, col);
          }
          if (i == S - 1 && r0 + 2 * S < w[c]) {  // this block's buffer is free: fetch the block after the next
            __syncwarp();
            issue_cols(c, b + 2);
          }
        }
      }
    }
    // drain: the last P items of the final pass
    if (maxw > 0) {
      const int r0 = ((maxw + S - 1) / S - 1) * S;
#pragma unroll
      for (int t = NI - P; t < NI; ++t) {
        const int mc = t % NCP, mi = t / NCP;
        if (r0 + mi < w[mc]) retire(mc, mi, xr[t % P]);
      }
    }
    return;
  }

  // ------------------------------- consumer -------------------------------
  const int c = warp;
  if (c >= ncons) return;
  const int slot = (s0 + c) * 32 + lane;
  const int row = Sv.slot_row[slot];
  const int len = Sv.slot_len[slot];
  const int wd = (int)((Sv.slice_ptr[s0 + c + 1] - Sv.slice_ptr[s0 + c]) >> 5);
  MC<K> acc = zero<K>();
  for (int r0 = 0; r0 < wd; r0 += S) {
    const uint32_t ph = (uint32_t)(r0 / S) & 1u;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const int r = r0 + i;
      if (r < wd) {
        const uint32_t full = bar0 + (c * S + i) * 8, empty = full + NC * S * 8;
        const unsigned char* stg = smem + (c * S + i) * STG;
        mbar_wait(full, ph);
        AVal<K, MX> a;
        if constexpr (MX) {
          a.a = reinterpret_cast<const double*>(stg)[lane];
        } else {
#pragma unroll
          for (int j = 0; j < K; ++j) a.a.c[j] = reinterpret_cast<const double*>(stg + j * 256)[lane];
        }
        MC<K> v;
        if constexpr (PB == 16) {
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const double2 t = reinterpret_cast<const double2*>(stg + A_BYTES + p * 512)[lane];
            v.c[2 * p] = t.x;
            v.c[2 * p + 1] = t.y;
          }
        } else {
#pragma unroll
          for (int p = 0; p < NP; ++p) v.c[p] = reinterpret_cast<const double*>(stg + A_BYTES + p * 256)[lane];
        }
        if (r < len) a.accumulate_lvl(acc, v);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty);
      }
    }
    acc = lvl_sweep(acc);
  }
  acc = canon(acc);
  if (row >= 0) store_aos<K>(y, row, acc);
}

}  // namespace ws
}  // namespace mpsg
