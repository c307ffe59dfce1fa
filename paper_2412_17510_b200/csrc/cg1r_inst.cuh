// cg1r_inst.cuh -- conjugate gradient with ONE reduction per iteration
// (Chronopoulos-Gear form), the variant the row-sharded solve uses.
//
// The reference's CG (krylov.hpp:238-281) needs two dot products per
// iteration with a vector update between them: <p,q> for alpha, then <r,r> of
// the updated residual.  On P GPUs each is an allgather + a dependent scalar
// step on the critical path (hard part 6).  The same Krylov
// iterates come out of the recurrences
//     p = r + beta p;   s = w + beta s   (s = A p without a product)
//     x = x + alpha p;  r = r - alpha s
//     w = A r                            (the iteration's SpMV)
//     gamma' = <r,r>;   delta = <w,r>    (ONE fused reduction, 2K doubles)
//     beta = gamma'/gamma;  sigma = delta - beta gamma'/alpha (= <p,Ap>);
//     alpha = gamma'/sigma
// (Chronopoulos & Gear 1989; parity for CG is stated in iterations, +-1%).
// The stop tests are the reference's record_step on sqrt(gamma'), the
// breakdown test its tiny(<p,Ap>) on sigma, with the reference's iteration
// count semantics.
//
// Sharded (mpsg_dcsr): per iteration one allgather of the rank partials
// (gamma', delta); the rank-ordered multi-component sum and the scalar
// recurrences run in the prologue of the NEXT update kernel, redundantly in
// every block (thread 0, broadcast through shared memory), so no one-thread
// launch sits between the collective and the update.  The scalar state is
// double-buffered (S[c] is read while block 0 writes S[c^1]).  r lives in the
// global-length buffer (its halo is exchanged before the SpMV).
#pragma once
#include "cg_inst.cuh"

namespace mpsg {

// One step of the scalar recurrences.  `prev` is the state before the step,
// (g, d) = (<r,r>, <w,r>) of the current residual; `writer` = the one thread
// that also records the step's history entries.
template <int K>
MPSG_DI CgState<K> cg1r_scalars(const CgState<K>& prev, bool init, const MC<K>& g, const MC<K>& d, bool writer) {
  CgState<K> o = prev;
  if (!init && prev.status != CG_RUNNING) return o;  // stopped earlier: carried forward unchanged
  bool cont = false;
  if (init) {
    // solver_init (krylov.hpp:187-197): history[0], converged-at-start
    const MC<K> rn = sqrt_mc(g);
    if (writer) o.history[0] = to_double(rn);
    o.k = 0;
    o.beta = zero<K>();
    if (less_equal(rn, prev.thr)) {
      o.status = 0;
    } else {
      o.status = CG_RUNNING;
      cont = true;
    }
  } else {
    const long long k = prev.k + 1;
    o.k = k;
    if (writer) {
#pragma unroll
      for (int j = 0; j < K; ++j) o.pend[k * K + j] = g.c[j];
    }
    if (surely_continues(g, prev.thr, prev.divergence_cap)) {
      cont = true;  // history[k] from pend after the loop (cg_history_kernel)
    } else {
      const MC<K> rn = sqrt_mc(g);
      const double rd = to_double(rn);
      if (writer) o.history[k] = rd;
      // record_step (krylov.hpp:205-213)
      if (!finite(rd)) {
        o.status = 2;
        o.reason = 2;
      } else if (less_equal(rn, prev.thr)) {
        o.status = 0;
      } else if (rd > prev.divergence_cap) {
        o.status = 3;
      } else {
        cont = true;
      }
    }
    if (cont) {
      o.beta = divide(g, prev.rho);
      if (k >= prev.max_iters) {
        o.status = 1;
        cont = false;
      }
    }
  }
  o.rho = g;
  if (cont) {
    // sigma = <p, A p> of the direction the next update builds
    const MC<K> sg = init ? d : sub(d, divide(mul(o.beta, g), prev.alpha));
    o.sigma = sg;
    const double sd = to_double(sg);
    if (!finite(sd) || fabs(sd) < prev.breakdown_floor) {  // krylov.hpp:250-254
      o.status = 2;
      o.reason = 1;
    } else {
      o.alpha = divide(g, sg);
    }
  }
  return o;
}

// Update kernel: p = r + beta p; s = w + beta s; x += alpha p; r -= alpha s.
// gathered != nullptr (sharded): the prologue folds the allgathered partials
// [rank][gamma K | delta K] into the new scalar state (see the header).
template <int K, bool F>
__global__ void __launch_bounds__(256) cg1r_update_kernel(CgState<K>* S, int c, int init, const double* gathered,
                                                          int nranks, int64_t n, double* x, double* r, double* p,
                                                          double* s, const double* w) {
  __shared__ MC<K> sh_ab[2];
  __shared__ int sh_status;
  if (threadIdx.x == 0) {
    if (gathered) {
      MC<K> g = zero<K>(), d = zero<K>();
      for (int q = 0; q < nranks; ++q) {
        g = add(g, load_aos_rw<K>(gathered, 2 * q));
        d = add(d, load_aos_rw<K>(gathered, 2 * q + 1));
      }
      const CgState<K> o = cg1r_scalars<K>(S[c ^ 1], init != 0, g, d, blockIdx.x == 0);
      if (blockIdx.x == 0) S[c] = o;
      sh_ab[0] = o.alpha;
      sh_ab[1] = o.beta;
      sh_status = o.status;
    } else {
      sh_ab[0] = S[c].alpha;
      sh_ab[1] = S[c].beta;
      sh_status = S[c].status;
    }
  }
  __syncthreads();
  if (sh_status != CG_RUNNING) return;
  const MC<K> alpha = sh_ab[0], beta = sh_ab[1], malpha = negate(alpha);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const MC<K> pi = pma<F>(load_aos_rw<K>(r, i), beta, load_aos_rw<K>(p, i));
    const MC<K> si = pma<F>(load_aos<K>(w, i), beta, load_aos_rw<K>(s, i));
    store_aos<K>(p, i, pi);
    store_aos<K>(s, i, si);
    store_aos<K>(x, i, pma<F>(load_aos_rw<K>(x, i), alpha, pi));
    store_aos<K>(r, i, pma<F>(load_aos_rw<K>(r, i), malpha, si));
  }
}

// The fused reduction (gamma', delta) = (<r,r>, <w,r>): fixed grid, fixed
// strides, fixed trees (as cg_reduce_kernel).  The last block either runs the
// scalar step (single GPU: S[c^1] = step(S[c])) or stores this rank's two
// totals in local_out (sharded).
template <int K, bool F>
__global__ void MPSG_DOT_LB cg1r_dots_kernel(CgState<K>* S, int c, int init, int gate, int64_t n, const double* r,
                                             const double* w, double* partial, double* local_out) {
  __shared__ MC<K> sh[DOT_THREADS / 32];
  __shared__ bool last;
  if (gate && S[c].status != CG_RUNNING) {
    // stopped: the state is carried forward so the final one is always S[c^1]
    if (!local_out && blockIdx.x == 0 && threadIdx.x == 0) S[c ^ 1] = S[c];
    return;
  }
  const int G = gridDim.x;
  const int64_t seg = (n + G - 1) / G;
  const int64_t lo = (int64_t)blockIdx.x * seg;
  const int64_t hi = (lo + seg < n) ? lo + seg : n;
  MC<K> ag = zero<K>(), ad = zero<K>();
  int64_t i = lo + threadIdx.x;
  MC<K> rn = zero<K>(), wn = zero<K>();
  if (i < hi) {
    rn = load_aos<K>(r, i);
    wn = load_aos<K>(w, i);
  }
  for (; i < hi; i += DOT_THREADS) {
    const MC<K> rr = rn, ww = wn;
    if (i + DOT_THREADS < hi) {
      rn = load_aos<K>(r, i + DOT_THREADS);
      wn = load_aos<K>(w, i + DOT_THREADS);
    }
    ag = pacc<F>(ag, rr, rr);
    ad = pacc<F>(ad, ww, rr);
  }
  const MC<K> bg = block_reduce<K, F>(ag, sh);
  __syncthreads();
  const MC<K> bd = block_reduce<K, F>(ad, sh);
  if (threadIdx.x == 0) {
    double* pp = partial + (int64_t)blockIdx.x * 2 * K;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      __stcg(pp + j, bg.c[j]);
      __stcg(pp + K + j, bd.c[j]);
    }
    __threadfence();
    last = (atomicAdd(&S[0].ticket, 1u) == (unsigned)(G - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int per = (G + DOT_THREADS - 1) / DOT_THREADS;
  MC<K> sg = zero<K>(), sd = zero<K>();
  for (int b = threadIdx.x * per; b < (threadIdx.x + 1) * per && b < G; ++b) {
    MC<K> pg, pd;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      pg.c[j] = __ldcg(partial + (int64_t)b * 2 * K + j);
      pd.c[j] = __ldcg(partial + (int64_t)b * 2 * K + K + j);
    }
    if constexpr (F && K >= 3 && MPSG_CG_LVL_TREE) {
      lvl_add(sg, pg);
      lvl_add(sd, pd);
    } else {
      sg = add(sg, pg);
      sd = add(sd, pd);
    }
  }
  __syncthreads();
  const MC<K> tg = block_reduce<K, F>(sg, sh);
  __syncthreads();
  const MC<K> td = block_reduce<K, F>(sd, sh);
  if (threadIdx.x == 0) {
    S[0].ticket = 0u;
    if (local_out) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        local_out[j] = tg.c[j];
        local_out[K + j] = td.c[j];
      }
    } else {
      const CgState<K> o = cg1r_scalars<K>(S[c], init != 0, tg, td, true);
      const unsigned keep = 0u;
      S[c ^ 1] = o;
      S[0].ticket = keep;
    }
  }
}

// Sharded: fold the last allgathered partials into the state (after a batch,
// before the host reads the status): S[c] = step(S[c^1]).
template <int K>
__global__ void cg1r_fold_kernel(CgState<K>* S, int c, int init, const double* gathered, int nranks) {
  MC<K> g = zero<K>(), d = zero<K>();
  for (int q = 0; q < nranks; ++q) {
    g = add(g, load_aos_rw<K>(gathered, 2 * q));
    d = add(d, load_aos_rw<K>(gathered, 2 * q + 1));
  }
  const CgState<K> o = cg1r_scalars<K>(S[c ^ 1], init != 0, g, d, true);
  const unsigned t = S[0].ticket;
  S[c] = o;
  S[0].ticket = t;
}

// S[1] = S[0] after the setup reductions (bnorm ... live in S[0])
template <int K>
__global__ void cg1r_copy_state_kernel(CgState<K>* S) {
  S[1] = S[0];
}

template <int K>
int cg1r_driver(mpsg_ctx* ctx, const mpsg_csr* A, const mpsg_dcsr* D, int order, const double* b_host,
                const double* x0, const mpsg_cg_config* cfg, double* x_out, double* history, int64_t history_cap,
                mpsg_cg_report* rep) {
  const double t0 = now_s();
  const int64_t n = A->nrows;  // local rows
  const int64_t nx = D ? D->nglobal : n;
  const int64_t off = D ? D->row_begin : 0;
  const int P = D ? D->comm->nranks : 1;
  const size_t vb = (size_t)n * K * sizeof(double);
  cudaStream_t st = ctx->stream;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  cudaGetLastError();
  const int64_t max_iters = cfg->max_iters;
  const char* efu = std::getenv("MPSG_CG_FUSED");
  const bool fused = order == MPSG_ORDER_FAST && K > 2 && !(efu && efu[0] == '0');
  double *b = nullptr, *x = nullptr, *rfull = nullptr, *p = nullptr, *s = nullptr, *w = nullptr, *part = nullptr,
         *hist = nullptr, *loc = nullptr, *gath = nullptr, *pend = nullptr;
  CgState<K>* S = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  auto cleanup = [&]() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    void* ps[] = {b, x, rfull, p, s, w, part, hist, loc, gath, S, pend};
    for (void* v : ps)
      if (v) cudaFree(v);
  };
  int rc = MPSG_OK;
#define CG_TRY(call)                                                                                    \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) {                                                                            \
      rc = fail(ctx, e_ == cudaErrorMemoryAllocation ? MPSG_E_OOM : MPSG_E_CUDA, "cg: %s: %s", #call,   \
                cudaGetErrorString(e_));                                                                \
      cleanup();                                                                                        \
      return rc;                                                                                        \
    }                                                                                                   \
  } while (0)
#define CG_RC(expr)      \
  do {                   \
    rc = (expr);         \
    if (rc != MPSG_OK) { \
      cleanup();         \
      return rc;         \
    }                    \
  } while (0)
  CG_TRY(cudaMalloc(&b, vb ? vb : 8));
  CG_TRY(cudaMalloc(&x, vb ? vb : 8));
  CG_TRY(cudaMalloc(&rfull, (size_t)std::max<int64_t>(nx, 1) * K * sizeof(double)));
  CG_TRY(cudaMalloc(&p, vb ? vb : 8));
  CG_TRY(cudaMalloc(&s, vb ? vb : 8));
  CG_TRY(cudaMalloc(&w, vb ? vb : 8));
  CG_TRY(cudaMalloc(&part, (size_t)DOT_MAX_BLOCKS * 2 * K * sizeof(double)));
  CG_TRY(cudaMalloc(&hist, (size_t)(max_iters + 1) * sizeof(double)));
  CG_TRY(cudaMalloc(&pend, (size_t)(max_iters + 1) * K * sizeof(double)));
  CG_TRY(cudaMalloc(&S, 2 * sizeof(CgState<K>)));
  if (D) {
    CG_TRY(cudaMalloc(&loc, (size_t)2 * K * sizeof(double)));
    CG_TRY(cudaMalloc(&gath, (size_t)P * 2 * K * sizeof(double)));
  }
  double* r = rfull + off * K;  // this rank's block of r

  auto occ_of = [](auto kern, int threads) {
    int o = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, 0);
    return std::max(o, 1);
  };
  auto wave = [&](int occ, int threads) {
    return (int)std::max<int64_t>(
        1, std::min<int64_t>({(int64_t)DOT_MAX_BLOCKS, (int64_t)sms * occ, (n + threads - 1) / threads}));
  };
  // setup reductions (bnorm, b - A x0) reuse the classic kernels on S[0]
  const int gset = wave(occ_of(cg_reduce_kernel<K, 0>, DOT_THREADS), DOT_THREADS);
  auto setup_reduce = [&](auto mode_tag, int post, const double* u, const double* v, double* xx) -> int {
    constexpr int MODE = decltype(mode_tag)::value;
    cg_reduce_kernel<K, MODE><<<gset, DOT_THREADS, 0, st>>>(S, post, n, u, v, xx, nullptr, part, 0,
                                                             D ? loc : nullptr);
    if (D) {
      int e = allgather_mc(D->comm, loc, gath, K, st);
      if (e) return e;
      cg_post_gathered_kernel<K><<<1, 1, 0, st>>>(S, post, gath, P, 0);
    }
    return cudaGetLastError() == cudaSuccess ? MPSG_OK : fail(ctx, MPSG_E_CUDA, "cg: reduction launch failed");
  };
  using Dot = std::integral_constant<int, 0>;
  using Res = std::integral_constant<int, 2>;
  auto apply = [&](double* out) -> int {  // out = A r over the global-length r
    if (D) return dist_spmv(D, order, rfull, nullptr, out, nullptr, st);
    return launch_spmv(ctx, A, order, rfull, nullptr, out, nullptr, st);
  };
  const int gdot = fused ? wave(occ_of(cg1r_dots_kernel<K, true>, DOT_THREADS), DOT_THREADS)
                         : wave(occ_of(cg1r_dots_kernel<K, false>, DOT_THREADS), DOT_THREADS);
  const int gupd = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 8, (n + 255) / 256));
  auto dots = [&](int c, int init, int gate) -> int {
    if (fused)
      cg1r_dots_kernel<K, true><<<gdot, DOT_THREADS, 0, st>>>(S, c, init, gate, n, r, w, part, D ? loc : nullptr);
    else
      cg1r_dots_kernel<K, false><<<gdot, DOT_THREADS, 0, st>>>(S, c, init, gate, n, r, w, part, D ? loc : nullptr);
    if (cudaGetLastError() != cudaSuccess) return fail(ctx, MPSG_E_CUDA, "cg: reduction launch failed");
    if (D) return allgather_mc(D->comm, loc, gath, 2 * K, st);
    return MPSG_OK;
  };
  auto update = [&](int c, int init) -> int {
    if (fused)
      cg1r_update_kernel<K, true><<<gupd, 256, 0, st>>>(S, c, init, D ? gath : nullptr, P, n, x, r, p, s, w);
    else
      cg1r_update_kernel<K, false><<<gupd, 256, 0, st>>>(S, c, init, D ? gath : nullptr, P, n, x, r, p, s, w);
    return cudaGetLastError() == cudaSuccess ? MPSG_OK : fail(ctx, MPSG_E_CUDA, "cg: update launch failed");
  };

  if (vb) CG_TRY(cudaMemcpyAsync(b, b_host, vb, cudaMemcpyHostToDevice, st));
  cg_init_state_kernel<K><<<1, 1, 0, st>>>(S, cfg->rel_tol, cfg->abs_tol, (long long)max_iters, hist, pend);
  CG_RC(setup_reduce(Dot{}, POST_BNORM, b, b, nullptr));
  if (x0) {
    // x = x0; r = b - A x0 (krylov.hpp:174-181)
    if (vb) {
      CG_TRY(cudaMemcpyAsync(x, x0, vb, cudaMemcpyHostToDevice, st));
      CG_TRY(cudaMemcpyAsync(r, x, vb, cudaMemcpyDeviceToDevice, st));
    }
    CG_RC(apply(w));
    CG_RC(setup_reduce(Res{}, POST_TRUE, b, nullptr, w));  // w = b - A x0 (the norm it leaves is overwritten later)
    if (vb) CG_TRY(cudaMemcpyAsync(r, w, vb, cudaMemcpyDeviceToDevice, st));
  } else {
    if (vb) {
      CG_TRY(cudaMemsetAsync(x, 0, vb, st));
      CG_TRY(cudaMemcpyAsync(r, b, vb, cudaMemcpyDeviceToDevice, st));
    }
  }
  if (vb) {
    CG_TRY(cudaMemsetAsync(p, 0, vb, st));
    CG_TRY(cudaMemsetAsync(s, 0, vb, st));
  }
  cg1r_copy_state_kernel<K><<<1, 1, 0, st>>>(S);
  // w0 = A r0; (gamma0, delta0); the first step's scalars land in S[1]
  CG_RC(apply(w));
  CG_RC(dots(0, 1, 0));
  if (D) cg1r_fold_kernel<K><<<1, 1, 0, st>>>(S, 1, 1, gath, P);
  CG_TRY(cudaGetLastError());
  CG_TRY(cudaStreamSynchronize(st));
  const double t_setup = now_s();

  // iteration with parity c: update from S[c] (sharded: recomputed from
  // S[c^1] + the gathered partials, idempotent), SpMV, fused reduction -> S[c^1]
  auto enqueue_iter = [&](int c) -> int {
    int e = update(c, 0);
    if (e) return e;
    if ((e = apply(w))) return e;
    return dots(c, 0, 1);
  };
  // the sharded update of the very first iteration re-derives S[1] from S[0]
  // with the init rule; afterwards every step uses the regular one
  int status = CG_RUNNING;
  {
    int hs;
    CG_TRY(cudaMemcpy(&hs, &S[1].status, sizeof(int), cudaMemcpyDeviceToHost));
    status = hs;
  }
  const int batch = cfg->check_every > 0 ? cfg->check_every : 32;
  long long done_k = 0;
  int c = 1;  // parity of the next iteration
  int gbatch = 0, gpar = -1;
  CG_TRY(cudaEventCreate(&ev0));
  CG_TRY(cudaEventCreate(&ev1));
  CG_TRY(cudaEventRecord(ev0, st));
  bool first = true;
  while (status == CG_RUNNING) {
    const long long remaining = max_iters - done_k;
    int nb = (int)std::min<long long>(batch, remaining);
    if (nb <= 0) break;
    if (first && D) {
      // first sharded iteration: its prologue folds (gamma0, delta0) with the init rule
      int e = MPSG_OK;
      if (fused)
        cg1r_update_kernel<K, true><<<gupd, 256, 0, st>>>(S, c, 1, gath, P, n, x, r, p, s, w);
      else
        cg1r_update_kernel<K, false><<<gupd, 256, 0, st>>>(S, c, 1, gath, P, n, x, r, p, s, w);
      CG_TRY(cudaGetLastError());
      if ((e = apply(w)) || (e = dots(c, 0, 1))) {
        cleanup();
        return e;
      }
      nb = 1;
    } else if (cfg->use_graph && !(D && D->comm->local)) {
      if (nb != gbatch || c != gpar) {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        gexec = nullptr;
        graph = nullptr;
        CG_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        int e = MPSG_OK;
        for (int i = 0; i < nb && e == MPSG_OK; ++i) e = enqueue_iter(c ^ (i & 1));
        cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (e != MPSG_OK || ce != cudaSuccess) {
          cleanup();
          return e != MPSG_OK ? e : fail(ctx, MPSG_E_CUDA, "cg: graph capture failed (%s)", cudaGetErrorString(ce));
        }
        CG_TRY(cudaGraphInstantiate(&gexec, graph, 0));
        gbatch = nb;
        gpar = c;
      }
      CG_TRY(cudaGraphLaunch(gexec, st));
    } else {
      for (int i = 0; i < nb; ++i) CG_RC(enqueue_iter(c ^ (i & 1)));
    }
    first = false;
    done_k += nb;
    c ^= (nb & 1);
    // the state after the batch is S[c] (sharded: fold the last partials first;
    // the next update's prologue recomputes the same values)
    if (D) cg1r_fold_kernel<K><<<1, 1, 0, st>>>(S, c, 0, gath, P);
    int hs;
    CG_TRY(cudaMemcpyAsync(&hs, &S[c].status, sizeof(int), cudaMemcpyDeviceToHost, st));
    CG_TRY(cudaStreamSynchronize(st));
    status = hs;
  }
  // deferred record_step values: history[k] = to_double(sqrt(<r,r>_k))
  cg_history_kernel<K><<<(int)std::min<int64_t>(148, (max_iters + 255) / 256), 256, 0, st>>>(S + c, pend, hist);
  CG_TRY(cudaGetLastError());
  CG_TRY(cudaEventRecord(ev1, st));
  CgState<K> hst;
  CG_TRY(cudaMemcpy(&hst, S + c, sizeof(hst), cudaMemcpyDeviceToHost));
  const double t_solve = now_s();
  float dev_ms = 0.f;
  cudaEventSynchronize(ev1);
  cudaEventElapsedTime(&dev_ms, ev0, ev1);
  const int64_t iters = hst.k;
  const int fstatus = hst.status == CG_RUNNING ? MPSG_MAX_ITERATIONS : hst.status;
  // final true residual ||b - A x|| (krylov.hpp:227-232): x through r's buffer
  if (vb) CG_TRY(cudaMemcpyAsync(r, x, vb, cudaMemcpyDeviceToDevice, st));
  CG_RC(apply(w));
  CG_RC(setup_reduce(Res{}, POST_TRUE, b, nullptr, w));
  double true_res = 0.0;
  CG_TRY(cudaMemcpyAsync(&true_res, &S[0].true_residual, sizeof(double), cudaMemcpyDeviceToHost, st));
  const int64_t nh = iters + 1;
  const int64_t ncopy = std::min<int64_t>(nh, history_cap);
  if (history && ncopy > 0)
    CG_TRY(cudaMemcpyAsync(history, hist, (size_t)ncopy * sizeof(double), cudaMemcpyDeviceToHost, st));
  double last_hist = 0.0;
  CG_TRY(cudaMemcpyAsync(&last_hist, hist + (nh - 1), sizeof(double), cudaMemcpyDeviceToHost, st));
  if (x_out && vb) CG_TRY(cudaMemcpyAsync(x_out, x, vb, cudaMemcpyDeviceToHost, st));
  CG_TRY(cudaStreamSynchronize(st));
  cleanup();

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
  const char* detail = "";
  if (fstatus == MPSG_BREAKDOWN) detail = hst.reason == 1 ? "cg: <p, Ap> vanished" : "cg: non-finite residual";
  std::snprintf(rep->detail, sizeof(rep->detail), "%s", detail);
  return MPSG_OK;
#undef CG_TRY
#undef CG_RC
}

// variant: MPSG_CG_AUTO = the reference's two-reduction iteration on one GPU,
// the one-reduction form when the rows are sharded over more than one rank.
inline bool cg_one_reduction(const mpsg_cg_config* cfg, const mpsg_dcsr* D) {
  if (cfg->variant == MPSG_CG_ONE_REDUCTION) return true;
  if (cfg->variant == MPSG_CG_CLASSIC) return false;
  return D && D->comm->nranks > 1;
}

template <int K>
int run_cg(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* b_host, const double* x0,
           const mpsg_cg_config* cfg, double* x_out, double* history, int64_t history_cap, mpsg_cg_report* rep) {
  if (cg_one_reduction(cfg, nullptr))
    return cg1r_driver<K>(ctx, A, nullptr, order, b_host, x0, cfg, x_out, history, history_cap, rep);
  return cg_driver<K>(ctx, A, nullptr, order, b_host, x0, cfg, x_out, history, history_cap, rep);
}

template <int K>
int run_dcg(mpsg_dcsr* D, int order, const double* b_host, const double* x0, const mpsg_cg_config* cfg,
            double* x_out, double* history, int64_t history_cap, mpsg_cg_report* rep) {
  if (cg_one_reduction(cfg, D))
    return cg1r_driver<K>(D->comm->ctx, D->local, D, order, b_host, x0, cfg, x_out, history, history_cap, rep);
  return cg_driver<K>(D->comm->ctx, D->local, D, order, b_host, x0, cfg, x_out, history, history_cap, rep);
}

}  // namespace mpsg

#define MPSG_INSTANTIATE_CG(K)                                                                            \
  template int mpsg::run_cg<K>(mpsg_ctx*, const mpsg_csr*, int, const double*, const double*,              \
                               const mpsg_cg_config*, double*, double*, int64_t, mpsg_cg_report*);         \
  template int mpsg::run_dcg<K>(mpsg_dcsr*, int, const double*, const double*, const mpsg_cg_config*,      \
                                double*, double*, int64_t, mpsg_cg_report*);
