// cg_inst.cuh -- device CG driver template, instantiated per K by cg_k{2,3,4}.cu.
//
// One driver for both the single-GPU solve (mpsg_cg) and the row-sharded
// multi-GPU solve (mpsg_dcg): with a distributed matrix D, vectors are this
// rank's row block, p lives in a global-length buffer whose halo is exchanged
// before every SpMV, and every dot product is reduced per rank, allgathered
// and summed in rank order (dist.h).  Without D the reductions finish in the
// last block of the reduction kernel itself.
#pragma once
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "cg_kernels.cuh"
#include "dist.h"
#include "internal.h"

namespace mpsg {

inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <int K>
int cg_driver(mpsg_ctx* ctx, const mpsg_csr* A, const mpsg_dcsr* D, int order, const double* b_host,
              const double* x0, const mpsg_cg_config* cfg, double* x_out, double* history, int64_t history_cap,
              mpsg_cg_report* rep) {
  const double t0 = now_s();
  const int64_t n = A->nrows;  // local rows
  const int64_t nx = D ? D->nglobal : n;
  const int64_t off = D ? D->row_begin : 0;
  const int P = D ? D->comm->nranks : 1;
  const size_t vb = (size_t)n * K * sizeof(double);
  cudaStream_t st = ctx->stream;
  // reduction grids: one resident wave (SMs x occupancy of the heaviest kernel)
  int sms = 148, occ = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cg_reduce_kernel<K, 1>, DOT_THREADS, 0);
  const char* genv = std::getenv("MPSG_CG_GRID");
  const int gpol = genv ? std::atoi(genv) : 1;
  const int64_t gwave = (int64_t)sms * std::max(occ, 1) * (gpol >= 2 ? gpol : 1);
  const int G = (int)std::max<int64_t>(
      1, std::min<int64_t>({(int64_t)DOT_MAX_BLOCKS, gpol == 0 ? (n + 2047) / 2048 : gwave,
                            (n + DOT_THREADS - 1) / DOT_THREADS}));
  const char* eoo = std::getenv("MPSG_CG_OWN_OCC");
  const bool own_occ = !(eoo && eoo[0] == '0');
  cudaGetLastError();
  double *b = nullptr, *x = nullptr, *r = nullptr, *pfull = nullptr, *q = nullptr, *part = nullptr,
         *hist = nullptr, *loc = nullptr, *gath = nullptr, *pend = nullptr;
  CgState<K>* dst = nullptr;
  const int64_t max_iters = cfg->max_iters;
  // FAST order: the iteration's vector updates and dots use the fused
  // product-accumulate too (MPSG_CG_FUSED=0 keeps the reference's add(mul))
  const char* efu = std::getenv("MPSG_CG_FUSED");
  const bool fused = order == MPSG_ORDER_FAST && K > 2 && !(efu && efu[0] == '0');
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;
  auto cleanup = [&]() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    void* ps[] = {b, x, r, pfull, q, part, hist, loc, gath, dst, pend};
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
#define CG_RC(expr)     \
  do {                  \
    rc = (expr);        \
    if (rc != MPSG_OK) { \
      cleanup();        \
      return rc;        \
    }                   \
  } while (0)
  CG_TRY(cudaMalloc(&b, vb ? vb : 8));
  CG_TRY(cudaMalloc(&x, vb ? vb : 8));
  CG_TRY(cudaMalloc(&r, vb ? vb : 8));
  CG_TRY(cudaMalloc(&pfull, (size_t)std::max<int64_t>(nx, 1) * K * sizeof(double)));
  CG_TRY(cudaMalloc(&q, vb ? vb : 8));
  CG_TRY(cudaMalloc(&part, (size_t)DOT_MAX_BLOCKS * K * sizeof(double)));
  CG_TRY(cudaMalloc(&hist, (size_t)(max_iters + 1) * sizeof(double)));
  CG_TRY(cudaMalloc(&pend, (size_t)(max_iters + 1) * K * sizeof(double)));
  CG_TRY(cudaMalloc(&dst, sizeof(CgState<K>)));
  if (D) {
    CG_TRY(cudaMalloc(&loc, (size_t)K * sizeof(double)));
    CG_TRY(cudaMalloc(&gath, (size_t)P * K * sizeof(double)));
  }
  double* p = pfull + off * K;  // this rank's block of p

  // one reduction: fused scalar step (single GPU) or partial -> allgather ->
  // rank-ordered sum -> scalar step (multi-GPU)
  auto reduce = [&](auto mode_tag, int post, const double* u, const double* v, double* xx, double* rr,
                    int gate) -> int {
    constexpr int MODE = decltype(mode_tag)::value;
    // this kernel's own resident wave (MPSG_CG_OWN_OCC=0: the shared grid G);
    // the occupancy is cached per instantiation, the grid follows n
    auto own_grid = [&](int occ_k) -> int {
      if (!own_occ) return G;
      const int64_t w = (int64_t)sms * std::max(occ_k, 1);
      return (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)DOT_MAX_BLOCKS, w,
                                                          (n + DOT_THREADS - 1) / DOT_THREADS}));
    };
    auto occ_of = [](auto kern) {
      int o = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, DOT_THREADS, 0);
      return o;
    };
    if (fused) {
      static const int of = occ_of(cg_reduce_kernel<K, MODE, true>);
      cg_reduce_kernel<K, MODE, true><<<own_grid(of), DOT_THREADS, 0, st>>>(dst, post, n, u, v, xx, rr, part,
                                                                             gate, D ? loc : nullptr);
    } else {
      static const int ou = occ_of(cg_reduce_kernel<K, MODE>);
      cg_reduce_kernel<K, MODE><<<own_grid(ou), DOT_THREADS, 0, st>>>(dst, post, n, u, v, xx, rr, part, gate,
                                                                      D ? loc : nullptr);
    }
    if (D) {
      int e = allgather_mc(D->comm, loc, gath, K, st);
      if (e) return e;
      cg_post_gathered_kernel<K><<<1, 1, 0, st>>>(dst, post, gath, P, gate);
    }
    return cudaGetLastError() == cudaSuccess ? MPSG_OK : fail(ctx, MPSG_E_CUDA, "cg: reduction launch failed");
  };
  using Dot = std::integral_constant<int, 0>;
  using Upd = std::integral_constant<int, 1>;
  using Res = std::integral_constant<int, 2>;
  // q = A p over the global-length p (halo first when sharded)
  auto apply = [&](double* out) -> int {
    if (D) return dist_spmv(D, order, pfull, nullptr, out, nullptr, st);  // halo overlapped with interior rows
    return launch_spmv(ctx, A, order, pfull, nullptr, out, nullptr, st);
  };

  if (vb) CG_TRY(cudaMemcpyAsync(b, b_host, vb, cudaMemcpyHostToDevice, st));
  cg_init_state_kernel<K><<<1, 1, 0, st>>>(dst, cfg->rel_tol, cfg->abs_tol, (long long)max_iters, hist, pend);
  // bnorm = norm2(b) (krylov.hpp:185)
  CG_RC(reduce(Dot{}, POST_BNORM, b, b, nullptr, nullptr, 0));
  if (x0) {
    // x = x0; r = b - A x0 (krylov.hpp:174-181)
    if (vb) {
      CG_TRY(cudaMemcpyAsync(x, x0, vb, cudaMemcpyHostToDevice, st));
      CG_TRY(cudaMemcpyAsync(p, x, vb, cudaMemcpyDeviceToDevice, st));
    }
    CG_RC(apply(r));
    CG_RC(reduce(Res{}, POST_R0, b, nullptr, r, nullptr, 0));
  } else {
    if (vb) {
      CG_TRY(cudaMemsetAsync(x, 0, vb, st));
      CG_TRY(cudaMemcpyAsync(r, b, vb, cudaMemcpyDeviceToDevice, st));
    }
    CG_RC(reduce(Dot{}, POST_R0, r, r, nullptr, nullptr, 0));
  }
  if (vb) CG_TRY(cudaMemcpyAsync(p, r, vb, cudaMemcpyDeviceToDevice, st));
  CG_TRY(cudaGetLastError());
  CG_TRY(cudaStreamSynchronize(st));
  const double t_setup = now_s();

  const int batch = cfg->check_every > 0 ? cfg->check_every : 32;
  const int ub = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n + 255) / 256));
  auto enqueue_iter = [&]() -> int {
    int e = apply(q);  // q = A p, sigma = <p, q> (krylov.hpp:248-249)
    if (e) return e;
    if ((e = reduce(Dot{}, POST_SIGMA, p, q, nullptr, nullptr, 1))) return e;
    if ((e = reduce(Upd{}, POST_RHO, p, q, x, r, 1))) return e;
    if (fused)
      cg_update_p_kernel<K, true><<<ub, 256, 0, st>>>(dst, n, r, p);
    else
      cg_update_p_kernel<K><<<ub, 256, 0, st>>>(dst, n, r, p);
    return cudaGetLastError() == cudaSuccess ? MPSG_OK : fail(ctx, MPSG_E_CUDA, "cg: update launch failed");
  };
  int status = CG_RUNNING;
  long long done_k = 0;
  {
    int hs;
    CG_TRY(cudaMemcpy(&hs, &dst->status, sizeof(int), cudaMemcpyDeviceToHost));
    status = hs;
  }
  int gbatch = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  CG_TRY(cudaEventCreate(&ev0));
  CG_TRY(cudaEventCreate(&ev1));
  CG_TRY(cudaEventRecord(ev0, st));
  while (status == CG_RUNNING) {
    long long remaining = max_iters - done_k;
    int nb = (int)std::min<long long>(batch, remaining);
    if (nb <= 0) break;
    // (a single-process group orders ranks with cross-stream events, which a
    // stream capture cannot record: no graphs there)
    if (cfg->use_graph && !(D && D->comm->local)) {
      if (nb != gbatch) {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        gexec = nullptr;
        graph = nullptr;
        CG_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        int e = MPSG_OK;
        for (int i = 0; i < nb && e == MPSG_OK; ++i) e = enqueue_iter();
        cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (e != MPSG_OK || ce != cudaSuccess) {
          cleanup();
          return e != MPSG_OK ? e : fail(ctx, MPSG_E_CUDA, "cg: graph capture failed (%s)", cudaGetErrorString(ce));
        }
        CG_TRY(cudaGraphInstantiate(&gexec, graph, 0));
        gbatch = nb;
      }
      CG_TRY(cudaGraphLaunch(gexec, st));
    } else {
      for (int i = 0; i < nb; ++i) CG_RC(enqueue_iter());
    }
    done_k += nb;
    int hs;
    CG_TRY(cudaMemcpyAsync(&hs, &dst->status, sizeof(int), cudaMemcpyDeviceToHost, st));
    CG_TRY(cudaStreamSynchronize(st));
    status = hs;
  }
  // deferred record_step values: history[k] = to_double(sqrt(<r,r>_k))
  cg_history_kernel<K><<<(int)std::min<int64_t>(148, (max_iters + 255) / 256), 256, 0, st>>>(dst, pend, hist);
  CG_TRY(cudaGetLastError());
  CG_TRY(cudaEventRecord(ev1, st));
  CgState<K> hst;
  CG_TRY(cudaMemcpy(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost));
  const double t_solve = now_s();
  float dev_ms = 0.f;
  cudaEventSynchronize(ev1);
  cudaEventElapsedTime(&dev_ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  // Iteration count semantics (krylov.hpp:251-253, 262-268, 276).
  const int64_t iters = hst.k;
  const int fstatus = hst.status == CG_RUNNING ? MPSG_MAX_ITERATIONS : hst.status;
  // final true residual ||b - A x|| (krylov.hpp:227-232): x through p's buffer
  if (vb) CG_TRY(cudaMemcpyAsync(p, x, vb, cudaMemcpyDeviceToDevice, st));
  CG_RC(apply(q));
  CG_RC(reduce(Res{}, POST_TRUE, b, nullptr, q, nullptr, 0));
  double true_res = 0.0;
  CG_TRY(cudaMemcpyAsync(&true_res, &dst->true_residual, sizeof(double), cudaMemcpyDeviceToHost, st));
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

}  // namespace mpsg
