// cg_kernels.cuh -- device-resident conjugate gradient (krylov.hpp:238-281).
//
// One CG iteration of the reference,
//     q = A p;  sigma = <p,q>;  breakdown if tiny(sigma);  alpha = rho/sigma;
//     x += alpha p;  r += (-alpha) q;  rho' = <r,r>;  |r| = sqrt(rho');
//     record / stop tests;  beta = rho'/rho;  p = r + beta p;  rho = rho'
// runs as four stream-ordered launches (SpMV, dot, fused x/r update + dot,
// p update) that never return to the host: the scalar recurrences (MC divide,
// sqrt, compare) and the stop tests run in the last block of each reduction
// and write a device-side state word the next launches read.  The host polls
// that word once per captured batch of iterations (CUDA graph).
//
// Dots use a fixed two-level tree (fixed grid, fixed per-thread strides,
// fixed block tree, fixed partial order), so results do not depend on
// scheduling; they are not the reference's sequential order (krylov.hpp:
// 122-128), which is why CG parity is stated in iterations and residuals.
#pragma once

#include "mc_arith.cuh"

namespace mpsg {

constexpr int CG_RUNNING = -1;

#ifndef MPSG_DOT_THREADS
#define MPSG_DOT_THREADS 256
#endif
#ifdef MPSG_DOT_MINB
#define MPSG_DOT_LB __launch_bounds__(DOT_THREADS, MPSG_DOT_MINB)
#else
#define MPSG_DOT_LB __launch_bounds__(DOT_THREADS)
#endif
#ifndef MPSG_CG_LVL_TREE
#define MPSG_CG_LVL_TREE 1
#endif
constexpr int DOT_THREADS = MPSG_DOT_THREADS;
constexpr int DOT_MAX_BLOCKS = 1024;

// Device-side solver state (one per solve).
template <int K>
struct CgState {
  MC<K> rho, sigma, alpha, beta, thr, bnorm, scratch;
  int status;         // CG_RUNNING or mpsg_solver_status
  int reason;         // 0 none, 1 <p,Ap> vanished, 2 non-finite residual
  long long k;        // completed iterations
  long long max_iters;
  double rel_tol, abs_tol, divergence_cap, breakdown_floor;
  double rhs_norm;
  double true_residual;
  double* history;    // [max_iters+1]
  double* pend;       // [max_iters+1][K]: <r,r> of every step; history = to_double(sqrt(pend))
  unsigned ticket;    // last-block arrival counter (self-resetting)
};

// acc + a*b: the reference's add(acc, mul(a, b)), or with the FAST order the
// fused form with one renormalisation (mc_arith.cuh fma_fast)
template <bool F, int K>
MPSG_DI MC<K> pma(const MC<K>& acc, const MC<K>& a, const MC<K>& b) {
  if constexpr (F)
    return fma_fast(acc, a, b);
  else
    return add(acc, mul(a, b));
}
// the same for a running dot accumulator (fma_acc: renorm sweep only)
template <bool F, int K>
MPSG_DI MC<K> pacc(const MC<K>& acc, const MC<K>& a, const MC<K>& b) {
  if constexpr (F)
    return fma_acc(acc, a, b);
  else
    return add(acc, mul(a, b));
}

enum DotPost {
  POST_BNORM = 0,  // bnorm = sqrt(<b,b>); threshold; caps
  POST_R0 = 1,     // <r,r>: rho; history[0]; converged-at-start test
  POST_SIGMA = 2,  // <p,q>: breakdown test; alpha
  POST_RHO = 3,    // <r,r> after the update: record_step; beta; rho
  POST_TRUE = 4    // ||b - A x||: final true residual
};

// F (FAST order, TD/QD): the tree combines on level sums (lvl_add), one sweep
// and renormalisation at the end -- the tree is the serial tail of every
// reduction kernel.
template <int K, bool F = false>
MPSG_DI MC<K> block_reduce(MC<K> v, MC<K>* sh) {
  constexpr bool LV = F && K >= 3 && MPSG_CG_LVL_TREE;
  // fixed xor tree inside each warp, then warp partials in warp order
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if constexpr (LV)
      lvl_add(v, shfl_xor(v, off));
    else
      v = add(v, shfl_xor(v, off));
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  // warp partials: a fixed xor tree in warp 0 (log2(warps) dependent adds)
  MC<K> s = zero<K>();
  if (w == 0) {
    const int nw = (int)(blockDim.x >> 5);
    if (lane < nw) s = sh[lane];
    for (int off = nw >> 1; off >= 1; off >>= 1) {
      if constexpr (LV)
        lvl_add(s, shfl_xor(s, off));
      else
        s = add(s, shfl_xor(s, off));
    }
    if constexpr (LV) s = canon(lvl_sweep(s));
  }
  return s;  // valid in thread 0
}

// The scalar tail of every reduction, run by thread 0 of the last block.
template <int K>
MPSG_DI void cg_post(CgState<K>* st, int post, const MC<K>& d) {
  if (post == POST_BNORM) {
    MC<K> bn = sqrt_mc(d);
    st->bnorm = bn;
    // threshold = bnorm * rel_tol + abs_tol (krylov.hpp:185-186)
    st->thr = add(mul_d(bn, st->rel_tol), from_double<K>(st->abs_tol));
    st->rhs_norm = to_double(bn);
    st->divergence_cap = 1e6 * st->rhs_norm + 1e6 * st->abs_tol;
    st->breakdown_floor = 1e-3 * st->abs_tol;
  } else if (post == POST_R0) {
    MC<K> rn = sqrt_mc(d);
    st->history[0] = to_double(rn);
    st->rho = d;
    st->k = 0;
    if (less_equal(rn, st->thr)) {  // krylov.hpp:193-197
      st->status = 0;
    } else {
      st->status = CG_RUNNING;
    }
  } else if (post == POST_SIGMA) {
    st->sigma = d;
    const double sd = to_double(d);
    if (!finite(sd) || fabs(sd) < st->breakdown_floor) {  // krylov.hpp:250-254, :234
      st->status = 2;
      st->reason = 1;
    } else {
      st->alpha = divide(st->rho, d);
    }
  } else if (post == POST_RHO) {
    const long long k = st->k + 1;
#pragma unroll
    for (int j = 0; j < K; ++j) st->pend[k * K + j] = d.c[j];
    st->k = k;
    if (surely_continues(d, st->thr, st->divergence_cap)) {
      // record_step continues for certain: history[k] is filled from pend by
      // cg_history_kernel after the loop (the square root is off the chain)
      st->beta = divide(d, st->rho);
      st->rho = d;
      if (k >= st->max_iters) st->status = 1;
      return;
    }
    MC<K> rn = sqrt_mc(d);
    const double rd = to_double(rn);
    st->history[k] = rd;
    // record_step (krylov.hpp:205-213)
    if (!finite(rd)) {
      st->status = 2;
      st->reason = 2;
    } else if (less_equal(rn, st->thr)) {
      st->status = 0;
    } else if (rd > st->divergence_cap) {
      st->status = 3;
    } else {
      st->beta = divide(d, st->rho);
      st->rho = d;
      if (k >= st->max_iters) st->status = 1;
    }
  } else if (post == POST_TRUE) {
    st->true_residual = to_double(sqrt_mc(d));
  }
}

// Block partial -> global partial[blockIdx]; the last block to arrive sums
// the G partials in a fixed order (thread t a contiguous run, then the block
// tree) and runs the scalar step (or, multi-GPU, stores this rank's total in
// local_out for the rank-ordered allgather sum).  Deterministic for a fixed
// grid size.
template <int K, int NT, bool F = false>
MPSG_DI void reduce_finish(CgState<K>* st, int post, MC<K> acc, double* partial, double* local_out, MC<K>* sh) {
  __shared__ bool last;
  const int G = gridDim.x;
  MC<K> bsum = block_reduce<K, F>(acc, sh);
  if (threadIdx.x == 0) {
    double* pp = partial + (int64_t)blockIdx.x * K;
#pragma unroll
    for (int j = 0; j < K; ++j) __stcg(pp + j, bsum.c[j]);
    __threadfence();
    last = (atomicAdd(&st->ticket, 1u) == (unsigned)(G - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int per = (G + NT - 1) / NT;
  MC<K> s = zero<K>();
  for (int i = threadIdx.x * per; i < (threadIdx.x + 1) * per && i < G; ++i) {
    MC<K> pv;
#pragma unroll
    for (int j = 0; j < K; ++j) pv.c[j] = __ldcg(partial + (int64_t)i * K + j);
    if constexpr (F && K >= 3 && MPSG_CG_LVL_TREE)
      lvl_add(s, pv);
    else
      s = add(s, pv);
  }
  __syncthreads();
  MC<K> tot = block_reduce<K, F>(s, sh);
  if (threadIdx.x == 0) {
    st->ticket = 0u;
    if (local_out) {
#pragma unroll
      for (int j = 0; j < K; ++j) local_out[j] = tot.c[j];
    } else {
      cg_post(st, post, tot);
    }
  }
}

// Generic reduction kernel.  MODE selects the per-element work:
//   0: d += u_i * v_i                                   (dots)
//   1: x_i += alpha p_i; r_i += (-alpha) q_i; d += r_i r_i (axpy pair + dot)
//   2: w_i = b_i - w_i; d += w_i w_i                    (true residual)
// The grid is sized to one resident wave (SMs x occupancy); each block owns a
// contiguous segment that its threads stride through (coalesced).
// local_out != nullptr (multi-GPU): see reduce_finish.
template <int K, int MODE, bool F = false>
__global__ void MPSG_DOT_LB cg_reduce_kernel(CgState<K>* st, int post, int64_t n,
                                                                const double* u, const double* v,
                                                                double* x, double* r, double* partial,
                                                                int gate, double* local_out) {
  __shared__ MC<K> sh[DOT_THREADS / 32];
  if (gate && st->status != CG_RUNNING) return;
  const int G = gridDim.x;
  const int64_t seg = (n + G - 1) / G;
  const int64_t lo = (int64_t)blockIdx.x * seg;
  const int64_t hi = (lo + seg < n) ? lo + seg : n;
  MC<K> acc = zero<K>();
  const MC<K> alpha = MODE == 1 ? st->alpha : zero<K>();
  const MC<K> malpha = negate(alpha);
  auto term = [&](int64_t i) -> MC<K> {
    if constexpr (MODE == 0) {
      return mul(load_aos_rw<K>(u, i), load_aos_rw<K>(v, i));
    } else if constexpr (MODE == 1) {
      // u = p, v = q; x, r updated in place (krylov.hpp:256-257: axpy = y + alpha*x)
      MC<K> xi = add(load_aos_rw<K>(x, i), mul(alpha, load_aos_rw<K>(u, i)));
      MC<K> ri = add(load_aos_rw<K>(r, i), mul(malpha, load_aos_rw<K>(v, i)));
      store_aos<K>(x, i, xi);
      store_aos<K>(r, i, ri);
      return mul(ri, ri);
    } else {
      // u = b, x = A x (overwritten with b - A x)
      MC<K> w = sub(load_aos_rw<K>(u, i), load_aos_rw<K>(x, i));
      store_aos<K>(x, i, w);
      return mul(w, w);
    }
  };
  if constexpr (MODE == 0) {
    // register double buffer: the next round's operands are in flight while
    // this round's product is accumulated
    int64_t i = lo + threadIdx.x;
    MC<K> un = zero<K>(), vn = zero<K>();
    if (i < hi) {
      un = load_aos<K>(u, i);
      vn = load_aos<K>(v, i);
    }
    for (; i < hi; i += DOT_THREADS) {
      const MC<K> uu = un, vv = vn;
      if (i + DOT_THREADS < hi) {
        un = load_aos<K>(u, i + DOT_THREADS);
        vn = load_aos<K>(v, i + DOT_THREADS);
      }
      acc = pacc<F>(acc, uu, vv);
    }
  } else if constexpr (MODE == 1) {
    int64_t i = lo + threadIdx.x;
    MC<K> pn = zero<K>(), qn = zero<K>(), xn = zero<K>(), rn = zero<K>();
    if (i < hi) {
      pn = load_aos<K>(u, i);
      qn = load_aos<K>(v, i);
      xn = load_aos_rw<K>(x, i);
      rn = load_aos_rw<K>(r, i);
    }
    for (; i < hi; i += DOT_THREADS) {
      const MC<K> pp = pn, qq = qn, xx = xn, rr = rn;
      if (i + DOT_THREADS < hi) {
        pn = load_aos<K>(u, i + DOT_THREADS);
        qn = load_aos<K>(v, i + DOT_THREADS);
        xn = load_aos_rw<K>(x, i + DOT_THREADS);
        rn = load_aos_rw<K>(r, i + DOT_THREADS);
      }
      const MC<K> xi = pma<F>(xx, alpha, pp);
      const MC<K> ri = pma<F>(rr, malpha, qq);
      store_aos<K>(x, i, xi);
      store_aos<K>(r, i, ri);
      acc = pacc<F>(acc, ri, ri);
    }
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += DOT_THREADS) acc = add(acc, term(i));
  }
  reduce_finish<K, DOT_THREADS, F>(st, post, acc, partial, local_out, sh);
}

// Rank-ordered multi-component sum of the allgathered partials, then the
// scalar step -- the same on every rank.
template <int K>
__global__ void cg_post_gathered_kernel(CgState<K>* st, int post, const double* gathered, int nranks, int gate) {
  if (gate && st->status != CG_RUNNING) return;
  MC<K> s = zero<K>();
  for (int q = 0; q < nranks; ++q) s = add(s, load_aos_rw<K>(gathered, q));
  cg_post(st, post, s);
}

// p = r + beta p (krylov.hpp:272)
template <int K, bool F = false>
__global__ void __launch_bounds__(256) cg_update_p_kernel(const CgState<K>* st, int64_t n,
                                                          const double* r, double* p) {
  if (st->status != CG_RUNNING) return;
  const MC<K> beta = st->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    store_aos<K>(p, i, pma<F>(load_aos_rw<K>(r, i), beta, load_aos_rw<K>(p, i)));
}

// Initial state: r = b (or b - A x0 computed by the caller), p = r.
// history[k] = to_double(sqrt(<r,r>_k)) for k = 1..kmax (record_step's value)
template <int K>
__global__ void cg_history_kernel(const CgState<K>* st, const double* pend, double* history) {
  const long long kmax = st->k;
  for (long long k = 1 + blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= kmax;
       k += (long long)gridDim.x * blockDim.x) {
    MC<K> d;
#pragma unroll
    for (int j = 0; j < K; ++j) d.c[j] = pend[k * K + j];
    history[k] = to_double(sqrt_mc(d));
  }
}

template <int K>
__global__ void cg_init_state_kernel(CgState<K>* st, double rel_tol, double abs_tol,
                                     long long max_iters, double* history, double* pend) {
  st->status = CG_RUNNING;
  st->reason = 0;
  st->k = 0;
  st->max_iters = max_iters;
  st->rel_tol = rel_tol;
  st->abs_tol = abs_tol;
  st->history = history;
  st->pend = pend;
  st->ticket = 0u;
  st->true_residual = 0.0;
}

}  // namespace mpsg
