// krylov_kernels.cuh -- device-resident Krylov engine for solve()
// (krylov.hpp:238-606: CG, BiCG, CGS, BiCGSTAB, GPBiCG).
//
// Every solver step is one of three generic launches over AoS vectors:
//   kr_reduce_kernel<K, M>  per-element body (vector updates + M product
//                           terms), M multi-component dot products reduced
//                           with a fixed tree, then a scalar `post` run by
//                           the last block to arrive (the method's scalar
//                           recurrences, breakdown tests and record_step);
//   kr_reduce_seq_kernel    the same body and post on ONE thread walking
//                           i = 0..n-1: every dot is the reference's
//                           sequential `acc = acc + u[i]*v[i]` (krylov.hpp:
//                           122-128), so with an exact SpMV order the whole
//                           solve reproduces the reference bit for bit;
//   kr_map_kernel           per-element body only.
// Bodies and posts are device lambdas written per method in krylov_inst.cuh
// next to the reference lines they restate.  The scalars live in KrState on
// the device; kernels read the state word and skip themselves once the solve
// has stopped, so batches of iterations can be captured in one CUDA graph and
// the host polls the state once per batch (as the CG driver does).
#pragma once

#include "mc_arith.cuh"

namespace mpsg {

constexpr int KR_RUNNING = -1;
constexpr int KR_HALF = -2;  // BiCGSTAB / GPBiCG half step converged: finish x, r, then Converged
constexpr int KR_THREADS = 256;
constexpr int KR_MAX_BLOCKS = 1024;

// Gates: which solver states a launch runs in.
enum KrGate { GATE_ALWAYS = 0, GATE_RUN = 1, GATE_RUN_HALF = 2 };

// The iteration scalars (read by the vector bodies, loaded once per thread).
template <int K>
struct KrScalars {
  MC<K> rho, alpha, beta, omega, zeta, eta;
  int half;   // the half step converged (status KR_HALF)
  int fused;  // FAST order with tree dots: product-accumulates with one renormalisation (fma_fast)
};

// One product term of a fused dot: the reduction adds a*b to its accumulator.
template <int K>
struct KrTerm {
  MC<K> a, b;
};

// x + a*b in the bodies: the reference's add(x, mul(a, b)), or fma_fast when
// the solve runs fused (never with the sequential, reference-exact dots).
template <int K>
MPSG_DI MC<K> pma(const KrScalars<K>& c, const MC<K>& x, const MC<K>& a, const MC<K>& b) {
  return c.fused ? fma_fast(x, a, b) : add(x, mul(a, b));
}

// Reason codes of a Breakdown (the detail text after "<method>: "), shared
// with the oracle (oracle/mpsoracle.c):
//   1 "<p, Ap> vanished"  2 "non-finite residual"  3 "<r~, r> vanished"
//   4 "<p~, Ap> vanished" 5 "<r~, Ap> vanished"    6 "<t, t> vanished"
//   7 "omega vanished"    8 "<At, At> vanished"    9 "zeta/eta system is singular"
//  10 "zeta vanished"
template <int K>
struct KrState {
  KrScalars<K> sc;
  MC<K> thr;          // rel_tol * ||b|| + abs_tol (krylov.hpp:185-186)
  int status;         // KR_RUNNING, KR_HALF or mpsg_solver_status
  int reason;
  long long k;        // completed iterations
  long long max_iters;
  double rel_tol, abs_tol, cap, floor;
  double rhs_norm;
  double true_residual;
  double* history;    // [max_iters + 1]
  double* pend;       // [max_iters + 1][K]: the squared norm of every recorded step
  unsigned ticket;    // last-block arrival counter (self-resetting)
};

MPSG_DI bool gate_open(int status, int gate) {
  return gate == GATE_ALWAYS || status == KR_RUNNING || (gate == GATE_RUN_HALF && status == KR_HALF);
}

// detail::tiny (krylov.hpp:234)
MPSG_DI bool kr_tiny(double v, double floor) { return !finite(v) || fabs(v) < floor; }

template <int K>
MPSG_DI void kr_break(KrState<K>* st, int reason) {
  st->status = MPSG_BREAKDOWN;
  st->reason = reason;
}

// record_step (krylov.hpp:203-213) + close_report's status mapping
// (:215-224): appends ||r_k|| for k = completed + 1; true while the
// iteration continues.
template <int K>
MPSG_DI void kr_pend(KrState<K>* st, long long k, const MC<K>& d) {
#pragma unroll
  for (int j = 0; j < K; ++j) st->pend[k * K + j] = d.c[j];
}

// record_step (krylov.hpp:203-213) + close_report's status mapping
// (:215-224) on ||r_k|| = sqrt(d), d = <r, r>, for k = completed + 1; true
// while the iteration continues.  When the outcome is certain
// (surely_continues) the multi-component square root is skipped here and the
// history entry is filled from pend by kr_history_kernel after the loop.
template <int K>
MPSG_DI bool kr_record(KrState<K>* st, const MC<K>& d) {
  const long long k = st->k + 1;
  kr_pend(st, k, d);
  st->k = k;
  if (surely_continues(d, st->thr, st->cap)) return true;
  const MC<K> rnorm = sqrt_call(d);
  const double rd = to_double(rnorm);
  st->history[k] = rd;
  if (!finite(rd)) {
    kr_break(st, 2);
    return false;
  }
  if (less_equal(rnorm, st->thr)) {
    st->status = MPSG_CONVERGED;
    return false;
  }
  if (rd > st->cap) {
    st->status = MPSG_DIVERGED;
    return false;
  }
  return true;
}

// The half-step test of BiCGSTAB / GPBiCG (krylov.hpp:423-424, 513-514):
// ||s|| = sqrt(d) <= threshold -> KR_HALF with the entry recorded.
template <int K>
MPSG_DI void kr_half_test(KrState<K>* st, const MC<K>& d) {
  if (surely_continues(d, st->thr, INFINITY)) return;
  const MC<K> sn = sqrt_call(d);
  if (less_equal(sn, st->thr)) {
    st->k += 1;
    kr_pend(st, st->k, d);
    st->history[st->k] = to_double(sn);
    st->status = KR_HALF;
    st->sc.half = 1;
  }
}

// history[k] = to_double(sqrt(pend[k])) for k = 1..completed (record_step's value)
template <int K>
__global__ void kr_history_kernel(const KrState<K>* st, double* history) {
  const long long kmax = st->k;
  const double* pend = st->pend;
  for (long long k = 1 + blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= kmax;
       k += (long long)gridDim.x * blockDim.x) {
    MC<K> d;
#pragma unroll
    for (int j = 0; j < K; ++j) d.c[j] = pend[k * K + j];
    history[k] = to_double(sqrt_mc(d));
  }
}

// End of an iteration that continues: the loop bound (krylov.hpp: `for (k =
// 1; k <= max_iters; ++k)`), then the next iteration's opening test on rho
// (tiny(<r~, r>), every method but CG).
template <int K>
MPSG_DI void kr_next(KrState<K>* st, bool check_rho) {
  if (st->k >= st->max_iters) {
    st->status = MPSG_MAX_ITERATIONS;
  } else if (check_rho && kr_tiny(to_double(st->sc.rho), st->floor)) {
    kr_break(st, 3);
  }
}

// lv (FAST order with tree dots, TD/QD): the tree combines run on level sums
// (lvl_add, mc_arith.cuh: QD 40 operations instead of the full add's 85) and
// are swept / renormalised once at the end -- the trees are the serial tail of
// every reduction kernel.
template <int K, int M>
MPSG_DI void block_reduce_m(MC<K> (&v)[M], MC<K>* sh, bool lv) {
  // fixed xor tree inside each warp, then warp partials in warp order
  if (lv) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
#pragma unroll 1
      for (int off = 16; off >= 1; off >>= 1) lvl_add(v[m], shfl_xor(v[m], off));
    }
  } else {
#pragma unroll
    for (int m = 0; m < M; ++m) v[m] = warp_tree(v[m]);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int m = 0; m < M; ++m) sh[w * M + m] = v[m];
  }
  __syncthreads();
  // warp partials: a fixed xor tree in warp 0 (log2(warps) dependent adds)
  if (w == 0) {
    const int nw = (int)(blockDim.x >> 5);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      MC<K> s = lane < nw ? sh[lane * M + m] : zero<K>();
      if (lv) {
        for (int off = nw >> 1; off >= 1; off >>= 1) lvl_add(s, shfl_xor(s, off));
        s = canon(lvl_sweep(s));
      } else {
        for (int off = nw >> 1; off >= 1; off >>= 1) s = add(s, shfl_xor(s, off));
      }
      v[m] = s;
    }
  }
  __syncthreads();
}

// Parallel reduction: G blocks own contiguous segments their threads stride
// through (coalesced); block partials go to partial[G][M][K]; the last block
// sums them in block order (thread t a contiguous run, then the block tree)
// and runs post(st, totals).  Deterministic for a fixed grid.
template <int K, int M, class Body, class Post>
__global__ void __launch_bounds__(KR_THREADS) kr_reduce_kernel(KrState<K>* st, int gate, int64_t n,
                                                               double* partial, Body body, Post post,
                                                               double* local_out) {
  __shared__ MC<K> sh[(KR_THREADS / 32) * M];
  __shared__ bool last;
  if (!gate_open(st->status, gate)) return;
  const KrScalars<K> sc = st->sc;
  const int G = gridDim.x;
  const int64_t seg = (n + G - 1) / G;
  const int64_t lo = (int64_t)blockIdx.x * seg;
  const int64_t hi = (lo + seg < n) ? lo + seg : n;
  MC<K> acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = zero<K>();
  for (int64_t i = lo + threadIdx.x; i < hi; i += KR_THREADS) {
    KrTerm<K> t[M];
    body(sc, i, t);
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] = sc.fused ? fma_acc(acc[m], t[m].a, t[m].b) : add(acc[m], mul(t[m].a, t[m].b));
  }
  const bool lv = sc.fused && K >= 3;
  block_reduce_m<K, M>(acc, sh, lv);
  if (threadIdx.x == 0) {
    double* pp = partial + (int64_t)blockIdx.x * M * K;
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int j = 0; j < K; ++j) __stcg(pp + m * K + j, acc[m].c[j]);
    __threadfence();
    last = (atomicAdd(&st->ticket, 1u) == (unsigned)(G - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int per = (G + KR_THREADS - 1) / KR_THREADS;
  MC<K> s[M];
#pragma unroll
  for (int m = 0; m < M; ++m) s[m] = zero<K>();
  for (int b = threadIdx.x * per; b < (threadIdx.x + 1) * per && b < G; ++b) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
      MC<K> pv;
#pragma unroll
      for (int j = 0; j < K; ++j) pv.c[j] = __ldcg(partial + ((int64_t)b * M + m) * K + j);
      if (lv)
        lvl_add(s[m], pv);
      else
        s[m] = add(s[m], pv);
    }
  }
  block_reduce_m<K, M>(s, sh, lv);
  if (threadIdx.x == 0) {
    st->ticket = 0u;
    if (local_out) {  // row-sharded: this rank's totals, summed across ranks by kr_post_gathered_kernel
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int j = 0; j < K; ++j) local_out[m * K + j] = s[m].c[j];
    } else {
      post(st, s);
    }
  }
}

// Sequential reduction (one thread, i ascending): the reference's dot order.
template <int K, int M, class Body, class Post>
__global__ void kr_reduce_seq_kernel(KrState<K>* st, int gate, int64_t n, Body body, Post post,
                                     double* local_out) {
  if (!gate_open(st->status, gate)) return;
  const KrScalars<K> sc = st->sc;
  MC<K> acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = zero<K>();
  for (int64_t i = 0; i < n; ++i) {
    KrTerm<K> t[M];
    body(sc, i, t);
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] = add(acc[m], mul(t[m].a, t[m].b));  // acc + u[i]*v[i] (krylov.hpp:126)
  }
  if (local_out) {
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int j = 0; j < K; ++j) local_out[m * K + j] = acc[m].c[j];
  } else {
    post(st, acc);
  }
}

// Row-sharded: the P ranks' totals (allgathered, rank-major [P][M][K]) summed
// in rank order with the multi-component add, then the post -- the same on
// every rank, so all ranks take the same decisions.
template <int K, int M, class Post>
__global__ void kr_post_gathered_kernel(KrState<K>* st, int gate, const double* gathered, int P, Post post) {
  if (!gate_open(st->status, gate)) return;
  MC<K> s[M];
#pragma unroll
  for (int m = 0; m < M; ++m) s[m] = zero<K>();
  for (int q = 0; q < P; ++q)
#pragma unroll
    for (int m = 0; m < M; ++m) s[m] = add(s[m], load_aos_rw<K>(gathered, (int64_t)q * M + m));
  post(st, s);
}

template <int K, class Body>
__global__ void __launch_bounds__(256) kr_map_kernel(const KrState<K>* st, int gate, int64_t n, Body body) {
  if (!gate_open(st->status, gate)) return;
  const KrScalars<K> sc = st->sc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    body(sc, i);
}

template <int K>
__global__ void kr_init_state_kernel(KrState<K>* st, double rel_tol, double abs_tol, long long max_iters,
                                     double* history, double* pend, int fused) {
  st->sc.rho = st->sc.alpha = st->sc.beta = st->sc.omega = st->sc.zeta = st->sc.eta = zero<K>();
  st->sc.half = 0;
  st->sc.fused = fused;
  st->thr = zero<K>();
  st->status = KR_RUNNING;
  st->reason = 0;
  st->k = 0;
  st->max_iters = max_iters;
  st->rel_tol = rel_tol;
  st->abs_tol = abs_tol;
  st->cap = st->floor = st->rhs_norm = st->true_residual = 0.0;
  st->history = history;
  st->pend = pend;
  st->ticket = 0u;
}

}  // namespace mpsg
