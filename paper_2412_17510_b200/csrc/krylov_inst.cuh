// krylov_inst.cuh -- device solve() driver (krylov.hpp:160-606), instantiated
// per K by krylov_k{2,3,4}.cu.
//
// Each method's iteration is written as the sequence of generic launches of
// krylov_kernels.cuh, with the per-element bodies and the scalar posts as
// device lambdas that restate the reference lines cited beside them op for op
// (operand order included: mul(a, b) is not symmetric at TD/QD).  Dots that
// the reference computes one after the other from vectors that are final at
// that point are fused into one pass (M accumulators); each accumulator is
// still its own dot, so the sequential mode stays bit-exact.
//
// Status flow: the posts set KrState::status exactly where the reference
// returns (close_report), with KrState::k = the iteration count the reference
// reports, so the residual history always has k + 1 entries.  The half-step
// exits of BiCGSTAB / GPBiCG (krylov.hpp:424-433, 514-522) pass through
// KR_HALF: the next launch finishes x and r and then marks Converged.
#pragma once
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "dist.h"
#include "internal.h"
#include "krylov_kernels.cuh"

namespace mpsg {

template <int K>
struct KrLauncher {
  mpsg_ctx* ctx;
  cudaStream_t st;
  KrState<K>* dst;
  int64_t n;
  double* partial;
  int G;     // reduction grid cap
  int ub;    // map grid
  bool seq;  // reference dot order (one thread)
  int sms;
  int occ_mode;  // blocks per SM of the reduction grid (0: the kernel's occupancy; MPSG_KR_OCC)
  const mpsg_dcsr* D;  // row-sharded: reductions finish across ranks
  double* loc;         // [5][K] this rank's totals
  double* gath;        // [P][5][K]

  int check(const char* what) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MPSG_OK : fail(ctx, MPSG_E_CUDA, "solve: %s launch failed: %s", what,
                                             cudaGetErrorString(e));
  }
  template <int M, class Body, class Post>
  int reduce(int gate, Body body, Post post) {
    if (seq) {
      kr_reduce_seq_kernel<K, M><<<1, 1, 0, st>>>(dst, gate, n, body, post, D ? loc : nullptr);
    } else {
      // one resident wave of this kernel (its own occupancy; a thread-safe
      // static: ranks of a single-process group solve on several host threads)
      static const int occ = [] {
        int o = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kr_reduce_kernel<K, M, Body, Post>, KR_THREADS, 0);
        return o < 1 ? 1 : o;
      }();
      const int o = occ_mode > 0 ? occ_mode : occ;
      const int g = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)G, (int64_t)sms * o));
      kr_reduce_kernel<K, M><<<g, KR_THREADS, 0, st>>>(dst, gate, n, partial, body, post, D ? loc : nullptr);
    }
    if (D) {
      int e = allgather_mc(D->comm, loc, gath, M * K, st);
      if (e) return e;
      kr_post_gathered_kernel<K, M><<<1, 1, 0, st>>>(dst, gate, gath, D->comm->nranks, post);
    }
    return check("reduction");
  }
  template <class Body>
  int map(int gate, Body body) {
    kr_map_kernel<K><<<ub, 256, 0, st>>>(dst, gate, n, body);
    return check("vector");
  }
};

inline double kr_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Vector slots (n x K doubles each).
enum KrVec { V_B, V_X, V_R, V_Q, V_RT, V_P, V_PT, V_QT, V_U, V_V, V_T, V_W, V_Z, V_Y, V_AT, V_D, V_COUNT };

// D != nullptr: row-sharded solve (mpsg_dsolve).  A is this rank's row block
// (global column indices), b / x0 / x_out its blocks; every vector is
// allocated global-length with this rank's rows at [row_begin, row_end), so
// the SpMV inputs get their halo exchanged in place (as the sharded CG), and
// every reduction is per-rank totals -> allgather -> rank-ordered sum -> post.
template <int K>
int krylov_driver(mpsg_ctx* ctx, const mpsg_csr* A, const mpsg_dcsr* D, const mpsg_solver_config* cfg, int order,
                  const double* b_host, const double* x0_host, double* x_out, double* history,
                  int64_t history_cap, mpsg_cg_report* rep) {
  const double t0 = kr_now();
  const int method = cfg->method;
  const int64_t n = A->nrows;  // local rows
  const int64_t nx = D ? D->nglobal : n;
  const int64_t off = D ? D->row_begin : 0;
  const int P = D ? D->comm->nranks : 1;
  const size_t vb = (size_t)n * K * sizeof(double);
  cudaStream_t st = ctx->stream;
  const bool seq = cfg->dot_order == MPSG_DOT_SEQUENTIAL;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)KR_MAX_BLOCKS, (n + KR_THREADS - 1) / KR_THREADS));
  const char* e_occ = std::getenv("MPSG_KR_OCC");
  const int occ_mode = e_occ ? std::atoi(e_occ) : 0;
  const int ub = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 8, (n + 255) / 256));
  const int64_t max_iters = cfg->max_iters;
  cudaGetLastError();

  double* V[V_COUNT] = {};
  double* Vbase[V_COUNT] = {};
  double *part = nullptr, *hist = nullptr, *pend = nullptr, *loc = nullptr, *gath = nullptr;
  KrState<K>* dst = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  const int saved_seg_T = ctx->seg_T;
  auto cleanup = [&]() {
    ctx->seg_T = saved_seg_T;
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (double* v : Vbase)
      if (v) cudaFree(v);
    if (loc) cudaFree(loc);
    if (gath) cudaFree(gath);
    if (part) cudaFree(part);
    if (hist) cudaFree(hist);
    if (pend) cudaFree(pend);
    if (dst) cudaFree(dst);
  };
  int rc = MPSG_OK;
#define KR_TRY(call)                                                                                   \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) {                                                                           \
      rc = fail(ctx, e_ == cudaErrorMemoryAllocation ? MPSG_E_OOM : MPSG_E_CUDA, "solve: %s: %s", #call, \
                cudaGetErrorString(e_));                                                               \
      cleanup();                                                                                       \
      return rc;                                                                                       \
    }                                                                                                  \
  } while (0)
#define KR_RC(expr)      \
  do {                   \
    rc = (expr);         \
    if (rc != MPSG_OK) { \
      cleanup();         \
      return rc;         \
    }                    \
  } while (0)

  // vectors each method touches
  static const int need[5][V_COUNT] = {
      //  B X R Q RT P PT QT U V T W Z Y AT D
      {1, 1, 1, 1, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // CG: p, q
      {1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0},  // BiCG: rt, p, pt, q, qt
      {1, 1, 1, 1, 1, 1, 0, 0, 1, 1, 1, 1, 0, 0, 0, 0},  // CGS: rt, u, p, q, v, t, w
      {1, 1, 1, 1, 1, 1, 0, 0, 0, 1, 1, 0, 0, 0, 0, 0},  // BiCGSTAB: rt, p, v, s (in Q), t
      {1, 1, 1, 1, 1, 1, 0, 0, 1, 0, 1, 1, 1, 1, 1, 1},  // GPBiCG: rt, p, Ap (in Q), t, w, u, z, y, At, d
  };
  const size_t vfull = (size_t)nx * K * sizeof(double);
  for (int i = 0; i < V_COUNT; ++i)
    if (need[method][i]) {
      KR_TRY(cudaMalloc(&Vbase[i], vfull ? vfull : 8));
      V[i] = Vbase[i] + off * K;
    }
  if (D) {
    KR_TRY(cudaMalloc(&loc, (size_t)5 * K * sizeof(double)));
    KR_TRY(cudaMalloc(&gath, (size_t)P * 5 * K * sizeof(double)));
  }
  KR_TRY(cudaMalloc(&part, (size_t)G * 5 * K * sizeof(double)));
  KR_TRY(cudaMalloc(&hist, (size_t)(max_iters + 1) * sizeof(double)));
  KR_TRY(cudaMalloc(&pend, (size_t)(max_iters + 1) * K * sizeof(double)));
  KR_TRY(cudaMalloc(&dst, sizeof(KrState<K>)));
  double *b = V[V_B], *x = V[V_X], *r = V[V_R], *q = V[V_Q], *rt = V[V_RT], *p = V[V_P], *pt = V[V_PT],
         *qt = V[V_QT], *u = V[V_U], *v = V[V_V], *t = V[V_T], *w = V[V_W], *z = V[V_Z], *y = V[V_Y],
         *at = V[V_AT], *dv = V[V_D];
  KrLauncher<K> L{ctx, st, dst, n, part, G, ub, seq, sms, occ_mode, D, loc, gath};
  const mpsg_csr* T = A->trans;
  // y = A v for a vector slot pointer v (this rank's block of a global-length
  // buffer): halo first when sharded (the SpMV reads global columns)
  auto apply = [&](double* in, double* out) -> int {
    double* full = in - off * K;
    if (D) return dist_spmv(D, order, full, nullptr, out, nullptr, st);  // halo overlapped with interior rows
    return launch_spmv(ctx, A, order, full, nullptr, out, nullptr, st);
  };
  // CsrOperator::apply_transposed = sptmv at `threads` (krylov.hpp:116-119)
  const int torder = order == MPSG_ORDER_FAST ? MPSG_ORDER_FAST : MPSG_ORDER_SCALAR;
  // the thread-segment bounds apply to the transposed launches only
  int seg_T = 1;
  auto apply_t = [&](const double* in, double* out) {
    ctx->seg_T = seg_T;
    const int e = launch_spmv(ctx, T, torder, in, nullptr, out, nullptr, st);
    ctx->seg_T = 1;
    return e;
  };
  if (method == MPSG_BICG) {
    if (D) {
      cleanup();
      return fail(ctx, MPSG_E_ARG, "bicg: the transposed product is not available on a row-sharded matrix");
    }
    if (!T) {
      cleanup();
      return fail(ctx, MPSG_E_ARG, "sptmv: matrix was uploaded without MPSG_CSR_TRANSPOSE");
    }
    KR_RC(set_segments(ctx, A, order, cfg->threads));
    seg_T = ctx->seg_T;
    ctx->seg_T = 1;
  }

  // ------------------------------------------------------------ solver_init
  // (krylov.hpp:160-201)
  if (vb) KR_TRY(cudaMemcpyAsync(b, b_host, vb, cudaMemcpyHostToDevice, st));
  // FAST order with tree dots: fused product-accumulates in the vector kernels
  // too (MPSG_KR_FUSED=0 keeps the reference's add(mul)); never with exact dots
  const char* efu = std::getenv("MPSG_KR_FUSED");
  const int fused = (!seq && order == MPSG_ORDER_FAST && K > 2 && !(efu && efu[0] == '0')) ? 1 : 0;
  kr_init_state_kernel<K><<<1, 1, 0, st>>>(dst, cfg->rel_tol, cfg->abs_tol, (long long)max_iters, hist, pend, fused);
  // bnorm = norm2(b); threshold, divergence cap, breakdown floor (:185-189)
  KR_RC(L.template reduce<1>(
      GATE_ALWAYS,
      [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
        const MC<K> bi = load_aos_rw<K>(b, i);
        d[0] = KrTerm<K>{bi, bi};
      },
      [=] __device__(KrState<K> * s, MC<K> * d) {
        const MC<K> bn = sqrt_call(d[0]);
        s->thr = add(mul_d(bn, s->rel_tol), from_double<K>(s->abs_tol));
        s->rhs_norm = to_double(bn);
        s->cap = 1e6 * s->rhs_norm + 1e6 * s->abs_tol;
        s->floor = 1e-3 * s->abs_tol;
      }));
  const bool has_x0 = x0_host != nullptr;
  if (has_x0) {
    // x = scalar_like(x0); r = b - A x (:174-181)
    if (vb) KR_TRY(cudaMemcpyAsync(x, x0_host, vb, cudaMemcpyHostToDevice, st));
    KR_RC(apply(x, q));
  } else if (vb) {
    KR_TRY(cudaMemsetAsync(x, 0, vb, st));
  }
  // r0 = norm2(r); history[0]; converged-at-start test (:191-197)
  KR_RC(L.template reduce<1>(
      GATE_ALWAYS,
      [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
        const MC<K> bi = load_aos_rw<K>(b, i);
        const MC<K> ri = has_x0 ? sub(bi, load_aos_rw<K>(q, i)) : bi;
        store_aos<K>(r, i, ri);
        d[0] = KrTerm<K>{ri, ri};
      },
      [=] __device__(KrState<K> * s, MC<K> * d) {
        const MC<K> rn = sqrt_call(d[0]);
        s->history[0] = to_double(rn);
        s->k = 0;
        s->status = less_equal(rn, s->thr) ? MPSG_CONVERGED : KR_RUNNING;
      }));
  // method set-up: r~ = p (= p~, = u) = r, zero recurrences; rho = <r~, r>
  if (method == MPSG_GPBICG && vb) {
    KR_TRY(cudaMemsetAsync(t, 0, vb, st));  // t_prev
    KR_TRY(cudaMemsetAsync(w, 0, vb, st));
    KR_TRY(cudaMemsetAsync(u, 0, vb, st));
    KR_TRY(cudaMemsetAsync(z, 0, vb, st));
  }
  const bool is_cg = method == MPSG_CG;
  KR_RC(L.template reduce<1>(
      GATE_RUN,
      [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
        const MC<K> ri = load_aos_rw<K>(r, i);
        store_aos<K>(p, i, ri);
        if (rt) store_aos<K>(rt, i, ri);
        if (pt) store_aos<K>(pt, i, ri);
        if (method == MPSG_CGS) store_aos<K>(u, i, ri);
        d[0] = KrTerm<K>{ri, ri};
      },
      [=] __device__(KrState<K> * s, MC<K> * d) {
        s->sc.rho = d[0];
        if (!is_cg && kr_tiny(to_double(d[0]), s->floor)) kr_break(s, 3);
      }));
  KR_TRY(cudaGetLastError());
  KR_TRY(cudaStreamSynchronize(st));
  const double t_setup = kr_now();

  // -------------------------------------------------------------- iterations
  // alpha = rho / sigma after a tiny(sigma) test with the method's reason
  auto post_alpha = [=] __device__(KrState<K> * s, MC<K> * d) {
    const int why = method == MPSG_CG ? 1 : method == MPSG_BICG ? 4 : 5;
    if (kr_tiny(to_double(d[0]), s->floor)) {
      kr_break(s, why);
    } else {
      s->sc.alpha = divide_call(s->sc.rho, d[0]);
    }
  };
  // record_step on ||r|| = sqrt(d[0]); rho' = d[1]; beta = rho'/rho (BiCG, CGS)
  auto post_rho_next = [=] __device__(KrState<K> * s, MC<K> * d) {
    if (!kr_record(s, d[0])) return;
    s->sc.beta = divide_call(d[1], s->sc.rho);
    s->sc.rho = d[1];
    kr_next(s, true);
  };

  auto enqueue_iter = [&]() -> int {
    int e = MPSG_OK;
    switch (method) {
      case MPSG_CG:  // krylov.hpp:246-273
        if ((e = apply(p, q))) return e;
        if ((e = L.template reduce<1>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
                   d[0] = KrTerm<K>{load_aos_rw<K>(p, i), load_aos_rw<K>(q, i)};  // sigma = <p, q>
                 },
                 post_alpha)))
          return e;
        if ((e = L.template reduce<1>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>& c, int64_t i, KrTerm<K>* d) {
                   const MC<K> xi = pma(c, load_aos_rw<K>(x, i), c.alpha, load_aos_rw<K>(p, i));
                   const MC<K> ri = pma(c, load_aos_rw<K>(r, i), negate(c.alpha), load_aos_rw<K>(q, i));
                   store_aos<K>(x, i, xi);
                   store_aos<K>(r, i, ri);
                   d[0] = KrTerm<K>{ri, ri};  // rho' = <r, r>
                 },
                 [=] __device__(KrState<K> * s, MC<K> * d) {
                   if (!kr_record(s, d[0])) return;
                   s->sc.beta = divide_call(d[0], s->sc.rho);
                   s->sc.rho = d[0];
                   kr_next(s, false);
                 })))
          return e;
        return L.map(GATE_RUN, [=] __device__(const KrScalars<K>& c, int64_t i) {
          store_aos<K>(p, i, pma(c, load_aos_rw<K>(r, i), c.beta, load_aos_rw<K>(p, i)));
        });

      case MPSG_BICG:  // krylov.hpp:293-330
        if ((e = apply(p, q))) return e;
        if ((e = apply_t(pt, qt))) return e;
        if ((e = L.template reduce<1>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
                   d[0] = KrTerm<K>{load_aos_rw<K>(pt, i), load_aos_rw<K>(q, i)};  // sigma = <p~, q>
                 },
                 post_alpha)))
          return e;
        if ((e = L.template reduce<2>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>& c, int64_t i, KrTerm<K>* d) {
                   const MC<K> ma = negate(c.alpha);
                   const MC<K> xi = pma(c, load_aos_rw<K>(x, i), c.alpha, load_aos_rw<K>(p, i));
                   const MC<K> ri = pma(c, load_aos_rw<K>(r, i), ma, load_aos_rw<K>(q, i));
                   const MC<K> rti = pma(c, load_aos_rw<K>(rt, i), ma, load_aos_rw<K>(qt, i));
                   store_aos<K>(x, i, xi);
                   store_aos<K>(r, i, ri);
                   store_aos<K>(rt, i, rti);
                   d[0] = KrTerm<K>{ri, ri};   // ||r||^2
                   d[1] = KrTerm<K>{rti, ri};  // rho' = <r~, r>
                 },
                 post_rho_next)))
          return e;
        return L.map(GATE_RUN, [=] __device__(const KrScalars<K>& c, int64_t i) {
          store_aos<K>(p, i, pma(c, load_aos_rw<K>(r, i), c.beta, load_aos_rw<K>(p, i)));
          store_aos<K>(pt, i, pma(c, load_aos_rw<K>(rt, i), c.beta, load_aos_rw<K>(pt, i)));
        });

      case MPSG_CGS:  // krylov.hpp:350-389
        if ((e = apply(p, v))) return e;
        if ((e = L.template reduce<1>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
                   d[0] = KrTerm<K>{load_aos_rw<K>(rt, i), load_aos_rw<K>(v, i)};  // sigma = <r~, v>
                 },
                 post_alpha)))
          return e;
        // q = u - alpha v; t = u + q; x += alpha t
        if ((e = L.map(GATE_RUN, [=] __device__(const KrScalars<K>& c, int64_t i) {
               const MC<K> ui = load_aos_rw<K>(u, i);
               const MC<K> qi = sub(ui, mul(c.alpha, load_aos_rw<K>(v, i)));
               const MC<K> ti = add(ui, qi);
               store_aos<K>(q, i, qi);
               store_aos<K>(t, i, ti);
               store_aos<K>(x, i, pma(c, load_aos_rw<K>(x, i), c.alpha, ti));
             })))
          return e;
        if ((e = apply(t, w))) return e;
        if ((e = L.template reduce<2>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>& c, int64_t i, KrTerm<K>* d) {
                   const MC<K> ri = pma(c, load_aos_rw<K>(r, i), negate(c.alpha), load_aos_rw<K>(w, i));
                   store_aos<K>(r, i, ri);
                   d[0] = KrTerm<K>{ri, ri};
                   d[1] = KrTerm<K>{load_aos_rw<K>(rt, i), ri};
                 },
                 post_rho_next)))
          return e;
        // u = r + beta q; p = u + beta (q + beta p)
        return L.map(GATE_RUN, [=] __device__(const KrScalars<K>& c, int64_t i) {
          const MC<K> qi = load_aos_rw<K>(q, i);
          const MC<K> ui = pma(c, load_aos_rw<K>(r, i), c.beta, qi);
          store_aos<K>(u, i, ui);
          store_aos<K>(p, i, pma(c, ui, c.beta, pma(c, qi, c.beta, load_aos_rw<K>(p, i))));
        });

      case MPSG_BICGSTAB: {  // krylov.hpp:407-469; s lives in q
        double* s_ = q;
        if ((e = apply(p, v))) return e;
        if ((e = L.template reduce<1>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
                   d[0] = KrTerm<K>{load_aos_rw<K>(rt, i), load_aos_rw<K>(v, i)};  // sigma = <r~, v>
                 },
                 post_alpha)))
          return e;
        // s = r - alpha v; half-step test on ||s|| (:421-433)
        if ((e = L.template reduce<1>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>& c, int64_t i, KrTerm<K>* d) {
                   const MC<K> si = pma(c, load_aos_rw<K>(r, i), negate(c.alpha), load_aos_rw<K>(v, i));
                   store_aos<K>(s_, i, si);
                   d[0] = KrTerm<K>{si, si};
                 },
                 [=] __device__(KrState<K> * s, MC<K> * d) { kr_half_test(s, d[0]); })))
          return e;
        if ((e = apply(s_, t))) return e;
        // tt = <t, t>; omega = <t, s> / tt (:434-446)
        if ((e = L.template reduce<2>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
                   const MC<K> ti = load_aos_rw<K>(t, i);
                   d[0] = KrTerm<K>{ti, ti};
                   d[1] = KrTerm<K>{ti, load_aos_rw<K>(s_, i)};
                 },
                 [=] __device__(KrState<K> * s, MC<K> * d) {
                   if (kr_tiny(to_double(d[0]), s->floor)) {
                     kr_break(s, 6);
                     return;
                   }
                   const MC<K> om = divide_call(d[1], d[0]);
                   s->sc.omega = om;
                   if (kr_tiny(to_double(om), s->floor)) kr_break(s, 7);
                 })))
          return e;
        // x += alpha p (+ omega s); r = s (- omega t); ||r||, <r~, r> (:426-427, 447-451)
        if ((e = L.template reduce<2>(
                 GATE_RUN_HALF,
                 [=] __device__(const KrScalars<K>& c, int64_t i, KrTerm<K>* d) {
                   const MC<K> si = load_aos_rw<K>(s_, i);
                   MC<K> xi = pma(c, load_aos_rw<K>(x, i), c.alpha, load_aos_rw<K>(p, i));
                   MC<K> ri = si;
                   if (!c.half) {
                     xi = pma(c, xi, c.omega, si);
                     ri = pma(c, si, negate(c.omega), load_aos_rw<K>(t, i));
                   }
                   store_aos<K>(x, i, xi);
                   store_aos<K>(r, i, ri);
                   d[0] = KrTerm<K>{ri, ri};
                   d[1] = KrTerm<K>{load_aos_rw<K>(rt, i), ri};
                 },
                 [=] __device__(KrState<K> * s, MC<K> * d) {
                   if (s->status == KR_HALF) {
                     s->status = MPSG_CONVERGED;
                     return;
                   }
                   if (!kr_record(s, d[0])) return;
                   // beta = (rho'/rho) (alpha/omega) (:464-465)
                   s->sc.beta = mul(divide_call(d[1], s->sc.rho), divide_call(s->sc.alpha, s->sc.omega));
                   s->sc.rho = d[1];
                   kr_next(s, true);
                 })))
          return e;
        // p = r + beta (p - omega v) (:466-467)
        return L.map(GATE_RUN, [=] __device__(const KrScalars<K>& c, int64_t i) {
          const MC<K> pv = sub(load_aos_rw<K>(p, i), mul(c.omega, load_aos_rw<K>(v, i)));
          store_aos<K>(p, i, pma(c, load_aos_rw<K>(r, i), c.beta, pv));
        });
      }

      case MPSG_GPBICG: {  // krylov.hpp:494-587; Ap lives in q, t and t_prev share t
        double* ap = q;
        if ((e = apply(p, ap))) return e;
        if ((e = L.template reduce<1>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
                   d[0] = KrTerm<K>{load_aos_rw<K>(rt, i), load_aos_rw<K>(ap, i)};  // sigma = <r~, Ap>
                 },
                 post_alpha)))
          return e;
        // d = t_prev - r; y = d + alpha (Ap - w); t = r - alpha Ap; half-step test (:507-522)
        if ((e = L.template reduce<1>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>& c, int64_t i, KrTerm<K>* d) {
                   const MC<K> ri = load_aos_rw<K>(r, i), api = load_aos_rw<K>(ap, i);
                   const MC<K> di = sub(load_aos_rw<K>(t, i), ri);
                   store_aos<K>(dv, i, di);
                   store_aos<K>(y, i, pma(c, di, c.alpha, sub(api, load_aos_rw<K>(w, i))));
                   const MC<K> ti = pma(c, ri, negate(c.alpha), api);
                   store_aos<K>(t, i, ti);
                   d[0] = KrTerm<K>{ti, ti};
                 },
                 [=] __device__(KrState<K> * s, MC<K> * d) { kr_half_test(s, d[0]); })))
          return e;
        if ((e = apply(t, at))) return e;
        // <At, t>, <At, At>, <y, y>, <y, At>, <y, t>; zeta, eta (:523-548)
        if ((e = L.template reduce<5>(
                 GATE_RUN,
                 [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
                   const MC<K> ati = load_aos_rw<K>(at, i), ti = load_aos_rw<K>(t, i), yi = load_aos_rw<K>(y, i);
                   d[0] = KrTerm<K>{ati, ti};
                   d[1] = KrTerm<K>{ati, ati};
                   d[2] = KrTerm<K>{yi, yi};
                   d[3] = KrTerm<K>{yi, ati};
                   d[4] = KrTerm<K>{yi, ti};
                 },
                 [=] __device__(KrState<K> * s, MC<K> * d) {
                   const MC<K> &att = d[0], &ata = d[1], &yy = d[2], &yat = d[3], &yt = d[4];
                   if (s->k + 1 == 1) {
                     if (kr_tiny(to_double(ata), s->floor)) {
                       kr_break(s, 8);
                       return;
                     }
                     s->sc.zeta = divide_call(att, ata);
                     s->sc.eta = zero<K>();
                   } else {
                     const MC<K> den = sub(mul(ata, yy), mul(yat, yat));
                     if (kr_tiny(to_double(den), s->floor * s->floor)) {
                       kr_break(s, 9);
                       return;
                     }
                     s->sc.zeta = divide_call(sub(mul(yy, att), mul(yt, yat)), den);
                     s->sc.eta = divide_call(sub(mul(ata, yt), mul(yat, att)), den);
                   }
                 })))
          return e;
        // u, z, x, r; ||r||, <r~, r> (:549-562); half step: x += alpha p, r = t
        if ((e = L.template reduce<2>(
                 GATE_RUN_HALF,
                 [=] __device__(const KrScalars<K>& c, int64_t i, KrTerm<K>* d) {
                   const MC<K> ti = load_aos_rw<K>(t, i);
                   MC<K> xi = pma(c, load_aos_rw<K>(x, i), c.alpha, load_aos_rw<K>(p, i));
                   MC<K> rn = ti;
                   if (!c.half) {
                     const MC<K> ri = load_aos_rw<K>(r, i);
                     const MC<K> ui = add(mul(c.zeta, load_aos_rw<K>(ap, i)),
                                          mul(c.eta, pma(c, load_aos_rw<K>(dv, i), c.beta, load_aos_rw<K>(u, i))));
                     const MC<K> zi = sub(add(mul(c.zeta, ri), mul(c.eta, load_aos_rw<K>(z, i))), mul(c.alpha, ui));
                     store_aos<K>(u, i, ui);
                     store_aos<K>(z, i, zi);
                     xi = add(xi, zi);
                     rn = pma(c, pma(c, ti, negate(c.eta), load_aos_rw<K>(y, i)), negate(c.zeta), load_aos_rw<K>(at, i));
                   }
                   store_aos<K>(x, i, xi);
                   store_aos<K>(r, i, rn);
                   d[0] = KrTerm<K>{rn, rn};
                   d[1] = KrTerm<K>{load_aos_rw<K>(rt, i), rn};
                 },
                 [=] __device__(KrState<K> * s, MC<K> * d) {
                   if (s->status == KR_HALF) {
                     s->status = MPSG_CONVERGED;
                     return;
                   }
                   if (!kr_record(s, d[0])) return;
                   if (kr_tiny(to_double(s->sc.zeta), s->floor)) {  // (:575-580), after record
                     kr_break(s, 10);
                     return;
                   }
                   s->sc.beta = mul(divide_call(s->sc.alpha, s->sc.zeta), divide_call(d[1], s->sc.rho));
                   s->sc.rho = d[1];
                   kr_next(s, true);
                 })))
          return e;
        // w = At + beta Ap; p = r + beta (p - u); t_prev = t (already in t) (:581-585)
        return L.map(GATE_RUN, [=] __device__(const KrScalars<K>& c, int64_t i) {
          store_aos<K>(w, i, pma(c, load_aos_rw<K>(at, i), c.beta, load_aos_rw<K>(ap, i)));
          store_aos<K>(p, i, pma(c, load_aos_rw<K>(r, i), c.beta, sub(load_aos_rw<K>(p, i), load_aos_rw<K>(u, i))));
        });
      }
    }
    return fail(ctx, MPSG_E_ARG, "solve: unknown method %d", method);
  };

  int status;
  KR_TRY(cudaMemcpy(&status, &dst->status, sizeof(int), cudaMemcpyDeviceToHost));
  const int batch = cfg->check_every > 0 ? cfg->check_every : 32;
  int gbatch = 0;
  long long done_k = 0;
  KR_TRY(cudaEventCreate(&ev0));
  KR_TRY(cudaEventCreate(&ev1));
  KR_TRY(cudaEventRecord(ev0, st));
  while (status == KR_RUNNING) {
    const long long remaining = max_iters - done_k;
    const int nb = (int)std::min<long long>(batch, remaining);
    if (nb <= 0) break;
    // (a single-process group orders ranks with cross-stream events, which a
    // stream capture cannot record: no graphs there)
    if (cfg->use_graph && !(D && D->comm->local)) {
      if (nb != gbatch) {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        gexec = nullptr;
        graph = nullptr;
        KR_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        int e = MPSG_OK;
        for (int i = 0; i < nb && e == MPSG_OK; ++i) e = enqueue_iter();
        cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (e != MPSG_OK || ce != cudaSuccess) {
          cleanup();
          return e != MPSG_OK ? e
                              : fail(ctx, MPSG_E_CUDA, "solve: graph capture failed (%s)", cudaGetErrorString(ce));
        }
        KR_TRY(cudaGraphInstantiate(&gexec, graph, 0));
        gbatch = nb;
      }
      KR_TRY(cudaGraphLaunch(gexec, st));
    } else {
      for (int i = 0; i < nb; ++i) KR_RC(enqueue_iter());
    }
    done_k += nb;
    KR_TRY(cudaMemcpyAsync(&status, &dst->status, sizeof(int), cudaMemcpyDeviceToHost, st));
    KR_TRY(cudaStreamSynchronize(st));
  }
  // deferred record_step values
  kr_history_kernel<K><<<(int)std::min<int64_t>(sms, (max_iters + 255) / 256), 256, 0, st>>>(dst, hist);
  KR_TRY(cudaGetLastError());
  KR_TRY(cudaEventRecord(ev1, st));
  KrState<K> hst;
  KR_TRY(cudaMemcpy(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost));
  const double t_solve = kr_now();
  float dev_ms = 0.f;
  cudaEventSynchronize(ev1);
  cudaEventElapsedTime(&dev_ms, ev0, ev1);
  const int64_t iters = hst.k;
  const int fstatus = hst.status < 0 ? MPSG_MAX_ITERATIONS : hst.status;

  // finish_true_residual: ||b - A x|| from a fresh product (krylov.hpp:226-232)
  KR_RC(apply(x, q));
  KR_RC(L.template reduce<1>(
      GATE_ALWAYS,
      [=] __device__(const KrScalars<K>&, int64_t i, KrTerm<K>* d) {
        const MC<K> wi = sub(load_aos_rw<K>(b, i), load_aos_rw<K>(q, i));
        d[0] = KrTerm<K>{wi, wi};
      },
      [=] __device__(KrState<K> * s, MC<K> * d) { s->true_residual = to_double(sqrt_call(d[0])); }));
  double true_res = 0.0;
  KR_TRY(cudaMemcpyAsync(&true_res, &dst->true_residual, sizeof(double), cudaMemcpyDeviceToHost, st));
  const int64_t nh = iters + 1;
  const int64_t ncopy = std::min<int64_t>(nh, history_cap);
  if (history && ncopy > 0)
    KR_TRY(cudaMemcpyAsync(history, hist, (size_t)ncopy * sizeof(double), cudaMemcpyDeviceToHost, st));
  double last_hist = 0.0;
  KR_TRY(cudaMemcpyAsync(&last_hist, hist + (nh - 1), sizeof(double), cudaMemcpyDeviceToHost, st));
  if (x_out && vb) KR_TRY(cudaMemcpyAsync(x_out, x, vb, cudaMemcpyDeviceToHost, st));
  KR_TRY(cudaStreamSynchronize(st));
  cleanup();

  static const char* names[5] = {"cg", "bicg", "cgs", "bicgstab", "gpbicg"};
  static const char* reasons[11] = {"",
                                    "<p, Ap> vanished",
                                    "non-finite residual",
                                    "<r~, r> vanished",
                                    "<p~, Ap> vanished",
                                    "<r~, Ap> vanished",
                                    "<t, t> vanished",
                                    "omega vanished",
                                    "<At, At> vanished",
                                    "zeta/eta system is singular",
                                    "zeta vanished"};
  std::memset(rep, 0, sizeof(*rep));
  rep->status = fstatus;
  rep->converged = fstatus == MPSG_CONVERGED;
  rep->iterations = iters;
  rep->history_len = ncopy;
  rep->rhs_norm = hst.rhs_norm;
  rep->final_recurrence_residual = last_hist;
  rep->final_true_residual = true_res;
  rep->setup_seconds = t_setup - t0;
  rep->solve_seconds = t_solve - t_setup;
  rep->device_seconds = dev_ms * 1e-3;
  if (fstatus == MPSG_BREAKDOWN && hst.reason > 0 && hst.reason <= 10)
    std::snprintf(rep->detail, sizeof(rep->detail), "%s: %s", names[method], reasons[hst.reason]);
  return MPSG_OK;
#undef KR_TRY
#undef KR_RC
}

}  // namespace mpsg

#define MPSG_INSTANTIATE_KRYLOV(K)                                                                         \
  template int mpsg::krylov_driver<K>(mpsg_ctx*, const mpsg_csr*, const mpsg_dcsr*, const mpsg_solver_config*, \
                                      int, const double*, const double*, double*, double*, int64_t,        \
                                      mpsg_cg_report*);
