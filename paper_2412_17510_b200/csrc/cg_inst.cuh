// cg_inst.cuh -- device CG driver template, instantiated per K by cg_k{2,3,4}.cu.
#pragma once
#include <algorithm>
#include <chrono>
#include <cstring>

#include "cg_kernels.cuh"
#include "internal.h"

namespace mpsg {

inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <int K>
int run_cg(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* b_host, const double* x0,
           const mpsg_cg_config* cfg, double* x_out, double* history, int64_t history_cap,
           mpsg_cg_report* rep) {
  const double t0 = now_s();
  const int64_t n = A->nrows;
  const size_t vb = (size_t)n * K * sizeof(double);
  cudaStream_t st = ctx->stream;
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(DOT_MAX_BLOCKS, (n + 2047) / 2048));
  double *b = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *part = nullptr,
         *hist = nullptr;
  CgState<K>* dst = nullptr;
  const int64_t max_iters = cfg->max_iters;
  auto cleanup = [&]() {
    void* ps[] = {b, x, r, p, q, part, hist, dst};
    for (void* v : ps)
      if (v) cudaFree(v);
  };
  int rc = MPSG_OK;
#define CG_TRY(call)                                                                         \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      rc = fail(ctx, e_ == cudaErrorMemoryAllocation ? MPSG_E_OOM : MPSG_E_CUDA, "cg: %s: %s", #call, \
                cudaGetErrorString(e_));                                                     \
      cleanup();                                                                             \
      return rc;                                                                             \
    }                                                                                        \
  } while (0)
  CG_TRY(cudaMalloc(&b, vb));
  CG_TRY(cudaMalloc(&x, vb));
  CG_TRY(cudaMalloc(&r, vb));
  CG_TRY(cudaMalloc(&p, vb));
  CG_TRY(cudaMalloc(&q, vb));
  CG_TRY(cudaMalloc(&part, (size_t)G * K * sizeof(double)));
  CG_TRY(cudaMalloc(&hist, (size_t)(max_iters + 1) * sizeof(double)));
  CG_TRY(cudaMalloc(&dst, sizeof(CgState<K>)));
  CG_TRY(cudaMemcpyAsync(b, b_host, vb, cudaMemcpyHostToDevice, st));
  cg_init_state_kernel<K><<<1, 1, 0, st>>>(dst, cfg->rel_tol, cfg->abs_tol, (long long)max_iters, hist);
  // bnorm = norm2(b) (krylov.hpp:185)
  cg_reduce_kernel<K, 0><<<G, DOT_THREADS, 0, st>>>(dst, POST_BNORM, n, b, b, nullptr, nullptr, part, 0);
  if (x0) {
    // x = x0; r = b - A x0 (krylov.hpp:174-181)
    CG_TRY(cudaMemcpyAsync(x, x0, vb, cudaMemcpyHostToDevice, st));
    if ((rc = launch_spmv(ctx, A, order, x, nullptr, r, nullptr, st)) != MPSG_OK) {
      cleanup();
      return rc;
    }
    cg_reduce_kernel<K, 2><<<G, DOT_THREADS, 0, st>>>(dst, POST_R0, n, b, nullptr, r, nullptr, part, 0);
  } else {
    CG_TRY(cudaMemsetAsync(x, 0, vb, st));
    CG_TRY(cudaMemcpyAsync(r, b, vb, cudaMemcpyDeviceToDevice, st));
    cg_reduce_kernel<K, 0><<<G, DOT_THREADS, 0, st>>>(dst, POST_R0, n, r, r, nullptr, nullptr, part, 0);
  }
  CG_TRY(cudaMemcpyAsync(p, r, vb, cudaMemcpyDeviceToDevice, st));
  CG_TRY(cudaGetLastError());
  CG_TRY(cudaStreamSynchronize(st));
  const double t_setup = now_s();

  const int batch = cfg->check_every > 0 ? cfg->check_every : 32;
  auto enqueue_iter = [&]() -> int {
    int e = launch_spmv(ctx, A, order, p, nullptr, q, nullptr, st);
    if (e) return e;
    cg_reduce_kernel<K, 0><<<G, DOT_THREADS, 0, st>>>(dst, POST_SIGMA, n, p, q, nullptr, nullptr, part, 1);
    cg_reduce_kernel<K, 1><<<G, DOT_THREADS, 0, st>>>(dst, POST_RHO, n, p, q, x, r, part, 1);
    const int ub = (int)std::min<int64_t>(148 * 8, (n + 255) / 256);
    cg_update_p_kernel<K><<<ub, 256, 0, st>>>(dst, n, r, p);
    return cudaGetLastError() == cudaSuccess ? MPSG_OK : MPSG_E_CUDA;
  };
  int status = CG_RUNNING;
  long long done_k = 0;
  {
    int hs;
    CG_TRY(cudaMemcpy(&hs, &dst->status, sizeof(int), cudaMemcpyDeviceToHost));
    status = hs;
  }
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;
  int gbatch = 0;
  while (status == CG_RUNNING) {
    long long remaining = max_iters - done_k;
    int nb = (int)std::min<long long>(batch, remaining);
    if (nb <= 0) break;
    if (cfg->use_graph) {
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
          return fail(ctx, MPSG_E_CUDA, "cg: graph capture failed (%s)", cudaGetErrorString(ce));
        }
        CG_TRY(cudaGraphInstantiate(&gexec, graph, 0));
        gbatch = nb;
      }
      CG_TRY(cudaGraphLaunch(gexec, st));
    } else {
      for (int i = 0; i < nb; ++i)
        if ((rc = enqueue_iter()) != MPSG_OK) {
          cleanup();
          return fail(ctx, rc, "cg: launch failed: %s", cudaGetErrorString(cudaGetLastError()));
        }
    }
    done_k += nb;
    int hs;
    CG_TRY(cudaMemcpyAsync(&hs, &dst->status, sizeof(int), cudaMemcpyDeviceToHost, st));
    CG_TRY(cudaStreamSynchronize(st));
    status = hs;
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  if (graph) cudaGraphDestroy(graph);
  CgState<K> hst;
  CG_TRY(cudaMemcpy(&hst, dst, sizeof(hst), cudaMemcpyDeviceToHost));
  const double t_solve = now_s();
  // Iteration count semantics (krylov.hpp:251-253, 262-268, 276).
  int64_t iters = hst.k;
  int fstatus = hst.status == CG_RUNNING ? MPSG_MAX_ITERATIONS : hst.status;
  if (hst.status == 2 && hst.reason == 1) iters = hst.k;  // breakdown before step k+1
  // final true residual ||b - A x|| (krylov.hpp:227-232)
  if ((rc = launch_spmv(ctx, A, order, x, nullptr, q, nullptr, st)) != MPSG_OK) {
    cleanup();
    return rc;
  }
  cg_reduce_kernel<K, 2><<<G, DOT_THREADS, 0, st>>>(dst, POST_TRUE, n, b, nullptr, q, nullptr, part, 0);
  CG_TRY(cudaGetLastError());
  double true_res = 0.0;
  CG_TRY(cudaMemcpyAsync(&true_res, &dst->true_residual, sizeof(double), cudaMemcpyDeviceToHost, st));
  const int64_t nh = iters + 1;
  const int64_t ncopy = std::min<int64_t>(nh, history_cap);
  if (history && ncopy > 0)
    CG_TRY(cudaMemcpyAsync(history, hist, (size_t)ncopy * sizeof(double), cudaMemcpyDeviceToHost, st));
  double last_hist = 0.0;
  CG_TRY(cudaMemcpyAsync(&last_hist, hist + (nh - 1), sizeof(double), cudaMemcpyDeviceToHost, st));
  if (x_out) CG_TRY(cudaMemcpyAsync(x_out, x, vb, cudaMemcpyDeviceToHost, st));
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
  const char* detail = "";
  if (fstatus == MPSG_BREAKDOWN) detail = hst.reason == 1 ? "cg: <p, Ap> vanished" : "cg: non-finite residual";
  std::snprintf(rep->detail, sizeof(rep->detail), "%s", detail);
  return MPSG_OK;
#undef CG_TRY
}


}  // namespace mpsg

#define MPSG_INSTANTIATE_CG(K)                                                                 \
  template int mpsg::run_cg<K>(mpsg_ctx*, const mpsg_csr*, int, const double*, const double*,   \
                               const mpsg_cg_config*, double*, double*, int64_t, mpsg_cg_report*);
