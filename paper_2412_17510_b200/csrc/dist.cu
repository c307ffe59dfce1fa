// dist.cu -- C ABI of the row-sharded multi-GPU layer (see dist.h).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include "dist.h"

using namespace mpsg;

namespace mpsg {

const NcclApi* NcclApi::get(std::string* err) {
  static NcclApi api;
  static bool ok = false;
  static std::string why;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    bool all = true;
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp) all = false;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.AllGather, "ncclAllGather");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    if (!all)
      why = "libnccl.so.2 lacks a required symbol";
    else
      ok = true;
  });
  if (!ok && err) *err = why;
  return ok ? &api : nullptr;
}

void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lk(m);
  const long gen = generation;
  if (++arrived == P) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return generation != gen; });
  }
}

namespace {
// One local-group "collective": every rank publishes (ptr, ready event);
// `pull(q, src)` enqueues this rank's copies out of rank q's buffer; then
// every rank waits until all copies out of its own buffer are done before it
// may overwrite it.
// A failure on this rank never skips a barrier: the other ranks are already
// inside the collective, so this rank goes through all three barriers and
// returns its first error at the end (the others complete normally).
template <class Pull>
int local_collective(const mpsg_comm* c, const void* mine, cudaStream_t st, Pull pull) {
  LocalGroup* g = c->local;
  const int r = c->rank;
  int rc = MPSG_OK;
  auto cu = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == MPSG_OK) rc = fail(c->ctx, MPSG_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  };
  cu(cudaSetDevice(c->ctx->device), "cudaSetDevice");
  g->ptr[(size_t)r] = mine;
  cu(cudaEventRecord(g->ready[(size_t)r], st), "cudaEventRecord");
  g->barrier();
  for (int q = 0; q < g->P && rc == MPSG_OK; ++q) {
    if (q == r) continue;
    cu(cudaStreamWaitEvent(st, g->ready[(size_t)q], 0), "cudaStreamWaitEvent");
    if (rc == MPSG_OK) rc = pull(q, g->ptr[(size_t)q]);
  }
  // recorded even after a failure: the producers wait on it before reuse
  cu(cudaEventRecord(g->consumed[(size_t)r], st), "cudaEventRecord");
  g->barrier();
  for (int q = 0; q < g->P; ++q)
    if (q != r) cu(cudaStreamWaitEvent(st, g->consumed[(size_t)q], 0), "cudaStreamWaitEvent");
  g->barrier();  // the events may be re-recorded by the next collective only now
  return rc;
}
}  // namespace

int halo_exchange(const mpsg_dcsr* A, double* xfull, cudaStream_t st) {
  const mpsg_comm* c = A->comm;
  if (c->nranks == 1) return MPSG_OK;
  const int K = A->K;
  if (c->local) {
    // every rank takes part (the plan is per pair; a rank with nothing to
    // receive still publishes its buffer for the others)
    return local_collective(c, xfull, st, [&](int q, const void* src) -> int {
      const int64_t rlo = A->recv[2 * q], rhi = A->recv[2 * q + 1];
      if (rhi > rlo)
        CUDA_TRY(c->ctx, cudaMemcpyAsync(xfull + rlo * K, static_cast<const double*>(src) + rlo * K,
                                         (size_t)(rhi - rlo) * K * sizeof(double), cudaMemcpyDefault, st));
      return MPSG_OK;
    });
  }
  // every rank enters the group (a rank that receives nothing may still send)
  NCCL_TRY(c, c->api->GroupStart());
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) continue;
    const int64_t slo = A->send[2 * q], shi = A->send[2 * q + 1];
    const int64_t rlo = A->recv[2 * q], rhi = A->recv[2 * q + 1];
    if (shi > slo)
      NCCL_TRY(c, c->api->Send(xfull + slo * K, (size_t)(shi - slo) * K, ncclDouble, q, c->comm, st));
    if (rhi > rlo)
      NCCL_TRY(c, c->api->Recv(xfull + rlo * K, (size_t)(rhi - rlo) * K, ncclDouble, q, c->comm, st));
  }
  NCCL_TRY(c, c->api->GroupEnd());
  return MPSG_OK;
}

int dist_spmv(const mpsg_dcsr* A, int order, double* xre, double* xim, double* yre, double* yim, cudaStream_t st) {
  mpsg_ctx* ctx = A->comm->ctx;
  int rc;
  if (!A->local_int) {
    if ((rc = halo_exchange(A, xre, st))) return rc;
    if (xim && (rc = halo_exchange(A, xim, st))) return rc;
    return launch_spmv(ctx, A->local, order, xre, xim, yre, yim, st, false);
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_side0, st));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_side0, 0));
  if ((rc = launch_spmv(ctx, A->local_int, order, xre, xim, yre, yim, ctx->side, false))) return rc;
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_side1, ctx->side));
  if ((rc = halo_exchange(A, xre, st))) return rc;
  if (xim && (rc = halo_exchange(A, xim, st))) return rc;
  if ((rc = launch_spmv(ctx, A->local_bnd, order, xre, xim, yre, yim, st, false))) return rc;
  CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_side1, 0));
  return MPSG_OK;
}

int allgather_mc(const mpsg_comm* c, const double* in, double* out, int K, cudaStream_t st) {
  if (c->nranks == 1 || c->local) {
    CUDA_TRY(c->ctx, cudaMemcpyAsync(out + (size_t)c->rank * K, in, (size_t)K * sizeof(double),
                                     cudaMemcpyDeviceToDevice, st));
    if (c->nranks == 1) return MPSG_OK;
    return local_collective(c, in, st, [&](int q, const void* src) -> int {
      CUDA_TRY(c->ctx, cudaMemcpyAsync(out + (size_t)q * K, src, (size_t)K * sizeof(double), cudaMemcpyDefault, st));
      return MPSG_OK;
    });
  }
  NCCL_TRY(c, c->api->AllGather(in, out, (size_t)K, ncclDouble, c->comm, st));
  return MPSG_OK;
}

int allgather_host(const mpsg_comm* c, const int64_t* mine, int64_t* all, int n) {
  const int P = c->nranks;
  if (P == 1) {
    std::copy(mine, mine + n, all);
    return MPSG_OK;
  }
  if (c->local) {
    LocalGroup* g = c->local;
    std::copy(mine, mine + n, g->meta.begin() + (size_t)c->rank * n);
    g->barrier();
    std::copy(g->meta.begin(), g->meta.begin() + (size_t)P * n, all);
    g->barrier();
    return MPSG_OK;
  }
  mpsg_ctx* ctx = c->ctx;
  int64_t* d = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&d, sizeof(int64_t) * n * (P + 1)));
  cudaStream_t st = ctx->stream;
  cudaMemcpyAsync(d, mine, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st);
  ncclResult_t r = c->api->AllGather(d, d + n, (size_t)n, ncclInt64, c->comm, st);
  cudaMemcpyAsync(all, d + n, sizeof(int64_t) * n * P, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(d);
  if (r != ncclSuccess) return fail(ctx, MPSG_E_NCCL, "setup allgather: %s", c->api->GetErrorString(r));
  if (e != cudaSuccess) return fail(ctx, MPSG_E_CUDA, "setup allgather: %s", cudaGetErrorString(e));
  return MPSG_OK;
}

}  // namespace mpsg

namespace {

void free_dcsr(mpsg_dcsr* A) {
  if (!A) return;
  mpsg_csr_destroy(A->local);
  mpsg_csr_destroy(A->local_int);
  mpsg_csr_destroy(A->local_bnd);
  for (double* p : {A->xfull[0], A->xfull[1], A->ybuf[0], A->ybuf[1]})
    if (p) cudaFree(p);
  delete A;
}

// Own block of a distributed vector into the global-length buffer (the halo
// follows inside dist_spmv).
int stage_own(mpsg_dcsr* A, const double* x_local, double* xfull, cudaMemcpyKind kind, cudaStream_t st) {
  const size_t b = (size_t)(A->row_end - A->row_begin) * A->K * sizeof(double);
  if (b) CUDA_TRY(A->comm->ctx, cudaMemcpyAsync(xfull + A->row_begin * A->K, x_local, b, kind, st));
  return MPSG_OK;
}

}  // namespace

extern "C" {

int mpsg_halo_plan(int nranks, int rank, const int64_t* bounds, const int64_t* need, int64_t* send,
                   int64_t* recv) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !bounds || !need || !send || !recv) return MPSG_E_ARG;
  for (int q = 0; q < nranks; ++q) {
    // what rank q reads of my rows / what I read of q's rows
    int64_t slo = std::max(need[2 * q], bounds[rank]), shi = std::min(need[2 * q + 1], bounds[rank + 1]);
    int64_t rlo = std::max(need[2 * rank], bounds[q]), rhi = std::min(need[2 * rank + 1], bounds[q + 1]);
    if (q == rank || shi <= slo) slo = shi = 0;
    if (q == rank || rhi <= rlo) rlo = rhi = 0;
    send[2 * q] = slo;
    send[2 * q + 1] = shi;
    recv[2 * q] = rlo;
    recv[2 * q + 1] = rhi;
  }
  return MPSG_OK;
}

int mpsg_comm_unique_id(unsigned char* id) {
  if (!id) return MPSG_E_ARG;
  std::string err;
  const NcclApi* api = NcclApi::get(&err);
  if (!api) return MPSG_E_NCCL;
  ncclUniqueId u;
  if (api->GetUniqueId(&u) != ncclSuccess) return MPSG_E_NCCL;
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return MPSG_OK;
}

int mpsg_comm_create(mpsg_ctx* ctx, int nranks, int rank, const unsigned char* id, mpsg_comm** out) {
  if (!ctx || !out || nranks < 1 || rank < 0 || rank >= nranks) return MPSG_E_ARG;
  *out = nullptr;
  auto* c = new mpsg_comm();
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  if (nranks > 1) {
    if (!id) {
      delete c;
      return fail(ctx, MPSG_E_ARG, "comm_create: a unique id is required for nranks > 1");
    }
    std::string err;
    c->api = NcclApi::get(&err);
    if (!c->api) {
      delete c;
      return fail(ctx, MPSG_E_NCCL, "comm_create: %s", err.c_str());
    }
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    cudaSetDevice(ctx->device);
    ncclResult_t r = c->api->CommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
      const char* s = c->api->GetErrorString(r);
      delete c;
      return fail(ctx, MPSG_E_NCCL, "ncclCommInitRank: %s", s);
    }
  }
  *out = c;
  return MPSG_OK;
}

int mpsg_comm_create_local(mpsg_ctx* const* ctxs, int nranks, mpsg_comm** out) {
  if (!ctxs || !out || nranks < 1) return MPSG_E_ARG;
  auto* g = new LocalGroup();
  g->P = nranks;
  g->ptr.assign((size_t)nranks, nullptr);
  g->ready.assign((size_t)nranks, nullptr);
  g->consumed.assign((size_t)nranks, nullptr);
  g->meta.assign((size_t)nranks * 8, 0);
  for (int r = 0; r < nranks; ++r) {
    out[r] = nullptr;
    if (!ctxs[r]) return MPSG_E_ARG;
  }
  for (int r = 0; r < nranks; ++r) {
    mpsg_ctx* ctx = ctxs[r];
    cudaSetDevice(ctx->device);
    if (cudaEventCreateWithFlags(&g->ready[(size_t)r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->consumed[(size_t)r], cudaEventDisableTiming) != cudaSuccess)
      return fail(ctx, MPSG_E_CUDA, "comm_create_local: event creation failed");
    for (int q = 0; q < nranks; ++q)  // peer access between distinct devices (best effort)
      if (ctxs[q]->device != ctx->device) {
        cudaDeviceEnablePeerAccess(ctxs[q]->device, 0);
        cudaGetLastError();
      }
    auto* c = new mpsg_comm();
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = r;
    c->local = g;
    out[r] = c;
  }
  g->refs = nranks;
  return MPSG_OK;
}

void mpsg_comm_destroy(mpsg_comm* c) {
  if (!c) return;
  if (c->comm && c->api) c->api->CommDestroy(c->comm);
  if (c->local) {
    mpsg::LocalGroup* g = c->local;
    bool last;
    {
      std::lock_guard<std::mutex> lk(g->m);
      last = --g->refs == 0;
    }
    if (last) {
      for (auto e : g->ready)
        if (e) cudaEventDestroy(e);
      for (auto e : g->consumed)
        if (e) cudaEventDestroy(e);
      delete g;
    }
  }
  delete c;
}

int mpsg_dcsr_upload(mpsg_comm* c, int K, int is_complex, int64_t nglobal, int64_t row_begin, int64_t row_end,
                     const int64_t* indptr, const int64_t* indices, const double* const* planes, mpsg_dcsr** out) {
  if (!c || !out || !indptr) return MPSG_E_ARG;
  *out = nullptr;
  mpsg_ctx* ctx = c->ctx;
  if (row_begin < 0 || row_end < row_begin || row_end > nglobal)
    return fail(ctx, MPSG_E_ARG, "dcsr_upload: bad row block [%lld, %lld) of %lld", (long long)row_begin,
                (long long)row_end, (long long)nglobal);
  const int64_t nloc = row_end - row_begin;
  auto* A = new mpsg_dcsr();
  std::unique_ptr<mpsg_dcsr, void (*)(mpsg_dcsr*)> holder(A, free_dcsr);
  A->comm = c;
  A->K = K;
  A->cplx = is_complex != 0;
  A->nglobal = nglobal;
  A->row_begin = row_begin;
  A->row_end = row_end;
  // Collective setup.  Every rank reaches both status exchanges below even if
  // its own local work failed (a bad column index, OOM): the exchange carries
  // a status word, so all ranks fail together instead of the healthy ones
  // blocking forever in a collective the failed rank never enters.
  int rc = mpsg_csr_upload(ctx, K, is_complex, nloc, nglobal, indptr, indices, planes, &A->local);
  // the column interval this rank reads (its own block is always local)
  int64_t lo = row_begin, hi = row_end;
  if (rc == MPSG_OK) {
    const int64_t nnz = indptr[nloc];
    for (int64_t k = 0; k < nnz; ++k) {
      lo = std::min(lo, indices[k]);
      hi = std::max(hi, indices[k] + 1);
    }
  }
  // every rank's row block, read interval and status (tiny allgather at setup)
  const int P = c->nranks;
  std::vector<int64_t> mine = {row_begin, row_end, lo, hi, (int64_t)rc}, all((size_t)5 * P);
  const std::string local_err = rc ? ctx->err : std::string();
  int grc = allgather_host(c, mine.data(), all.data(), 5);
  if (grc) return grc;
  for (int q = 0; q < P; ++q)
    if (all[5 * q + 4] != MPSG_OK) {
      if (q == c->rank) return fail(ctx, rc, "%s", local_err.c_str());
      return fail(ctx, (int)all[5 * q + 4], "dcsr_upload: rank %d failed its local upload (status %lld)", q,
                  (long long)all[5 * q + 4]);
    }
  A->bounds.assign((size_t)P + 1, 0);
  A->need.assign((size_t)2 * P, 0);
  for (int q = 0; q < P; ++q) {
    if (all[5 * q] != A->bounds[q])
      return fail(ctx, MPSG_E_ARG, "dcsr_upload: row blocks are not contiguous in rank order");
    A->bounds[q + 1] = all[5 * q + 1];
    A->need[2 * q] = all[5 * q + 2];
    A->need[2 * q + 1] = all[5 * q + 3];
  }
  if (A->bounds[P] != nglobal) return fail(ctx, MPSG_E_ARG, "dcsr_upload: row blocks do not cover the matrix");
  A->send.assign((size_t)2 * P, 0);
  A->recv.assign((size_t)2 * P, 0);
  mpsg_halo_plan(P, c->rank, A->bounds.data(), A->need.data(), A->send.data(), A->recv.data());
  for (int q = 0; q < P; ++q) A->halo_rows += A->recv[2 * q + 1] - A->recv[2 * q];
  // interior / boundary split for the halo overlap (MPSG_HALO_OVERLAP=0 disables)
  const char* eo = std::getenv("MPSG_HALO_OVERLAP");
  if (P > 1 && (!eo || eo[0] != '0') && A->halo_rows > 0) {
    std::vector<int> rint, rbnd;
    for (int64_t i = 0; i < nloc; ++i) {
      bool inside = true;
      for (int64_t k = indptr[i]; k < indptr[i + 1] && inside; ++k)
        inside = indices[k] >= row_begin && indices[k] < row_end;
      (inside ? rint : rbnd).push_back((int)i);
    }
    if (!rint.empty() && !rbnd.empty()) {
      const int np = (A->cplx ? 2 : 1) * K;
      auto sub = [&](const std::vector<int>& rows, mpsg_csr** out_csr) -> int {
        std::vector<int64_t> sp(rows.size() + 1, 0), si;
        for (size_t r = 0; r < rows.size(); ++r) sp[r + 1] = sp[r] + (indptr[rows[r] + 1] - indptr[rows[r]]);
        si.reserve((size_t)sp.back());
        std::vector<std::vector<double>> pl((size_t)np);
        for (auto& v : pl) v.reserve((size_t)sp.back());
        for (int row : rows)
          for (int64_t k = indptr[row]; k < indptr[row + 1]; ++k) {
            si.push_back(indices[k]);
            for (int j = 0; j < np; ++j) pl[(size_t)j].push_back(planes[j][k]);
          }
        std::vector<const double*> pp((size_t)np);
        for (int j = 0; j < np; ++j) pp[(size_t)j] = pl[(size_t)j].data();
        int e = mpsg_csr_upload(ctx, K, is_complex, (int64_t)rows.size(), nglobal, sp.data(), si.data(), pp.data(),
                                out_csr);
        if (e) return e;
        return remap_rows(ctx, *out_csr, rows);
      };
      rc = sub(rint, &A->local_int);
      if (rc == MPSG_OK) rc = sub(rbnd, &A->local_bnd);
      A->n_interior = (int64_t)rint.size();
    }
  }
  const size_t xb = (size_t)std::max<int64_t>(nglobal, 1) * K * sizeof(double);
  for (int j = 0; j < (A->cplx ? 2 : 1) && rc == MPSG_OK; ++j) {
    cudaError_t e = cudaMalloc(&A->xfull[j], xb);
    if (e == cudaSuccess) e = cudaMemset(A->xfull[j], 0, xb);
    if (e != cudaSuccess) rc = fail(ctx, MPSG_E_CUDA, "dcsr_upload: %s", cudaGetErrorString(e));
  }
  // second status exchange: the local work after the first one may have failed
  std::vector<int64_t> st1 = {(int64_t)rc}, st_all((size_t)P);
  const std::string local_err2 = rc ? ctx->err : std::string();
  if ((grc = allgather_host(c, st1.data(), st_all.data(), 1))) return grc;
  for (int q = 0; q < P; ++q)
    if (st_all[(size_t)q] != MPSG_OK) {
      if (q == c->rank) return fail(ctx, rc, "%s", local_err2.c_str());
      return fail(ctx, (int)st_all[(size_t)q], "dcsr_upload: rank %d failed its local setup (status %lld)", q,
                  (long long)st_all[(size_t)q]);
    }
  *out = holder.release();
  return MPSG_OK;
}

void mpsg_dcsr_destroy(mpsg_dcsr* A) { free_dcsr(A); }

int mpsg_dcsr_info(const mpsg_dcsr* A, int64_t* bounds, int64_t* halo_rows) {
  if (!A) return MPSG_E_ARG;
  if (bounds) std::copy(A->bounds.begin(), A->bounds.end(), bounds);
  if (halo_rows) *halo_rows = A->halo_rows;
  return MPSG_OK;
}

int mpsg_dcsr_interior_rows(const mpsg_dcsr* A, int64_t* interior_rows) {
  if (!A || !interior_rows) return MPSG_E_ARG;
  *interior_rows = A->n_interior;
  return MPSG_OK;
}

int mpsg_dspmv_dev(mpsg_dcsr* A, int order, const double* d_x_local, double* d_y_local, void* stream) {
  if (!A) return MPSG_E_ARG;
  if (A->cplx) return fail(A->comm->ctx, MPSG_E_ARG, "dspmv: matrix is complex, use mpsg_dspmv_complex_dev");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : A->comm->ctx->stream;
  int rc = stage_own(A, d_x_local, A->xfull[0], cudaMemcpyDeviceToDevice, st);
  if (rc) return rc;
  return dist_spmv(A, order, A->xfull[0], nullptr, d_y_local, nullptr, st);
}

int mpsg_dspmv_complex_dev(mpsg_dcsr* A, int order, const double* d_xr_local, const double* d_xi_local,
                           double* d_yr_local, double* d_yi_local, void* stream) {
  if (!A) return MPSG_E_ARG;
  if (!A->cplx) return fail(A->comm->ctx, MPSG_E_ARG, "dspmv_complex: matrix is real");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : A->comm->ctx->stream;
  int rc = stage_own(A, d_xr_local, A->xfull[0], cudaMemcpyDeviceToDevice, st);
  if (!rc) rc = stage_own(A, d_xi_local, A->xfull[1], cudaMemcpyDeviceToDevice, st);
  if (rc) return rc;
  return dist_spmv(A, order, A->xfull[0], A->xfull[1], d_yr_local, d_yi_local, st);
}

int mpsg_dspmv(mpsg_dcsr* A, int order, const double* x_local, double* y_local) {
  if (!A) return MPSG_E_ARG;
  mpsg_ctx* ctx = A->comm->ctx;
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "dspmv: matrix is complex, use mpsg_dspmv_complex_dev");
  const int64_t nloc = A->row_end - A->row_begin;
  const size_t b = (size_t)nloc * A->K * sizeof(double);
  const int ns = A->cplx ? 2 : 1;
  for (int j = 0; j < ns; ++j)
    if (!A->ybuf[j]) CUDA_TRY(ctx, cudaMalloc(&A->ybuf[j], b ? b : 8));
  cudaStream_t st = ctx->stream;
  int rc = stage_own(A, x_local, A->xfull[0], cudaMemcpyHostToDevice, st);
  if (rc) return rc;
  if ((rc = dist_spmv(A, order, A->xfull[0], nullptr, A->ybuf[0], nullptr, st))) return rc;
  if (b) CUDA_TRY(ctx, cudaMemcpyAsync(y_local, A->ybuf[0], b, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MPSG_OK;
}

int mpsg_dcg(mpsg_dcsr* A, int order, const double* b_local, const double* x0_local, const mpsg_cg_config* cfg,
             double* x_out_local, double* history, int64_t history_cap, mpsg_cg_report* report) {
  if (!A || !cfg || !report || (!b_local && A->row_end > A->row_begin)) return MPSG_E_ARG;
  mpsg_ctx* ctx = A->comm->ctx;
  if (!(cfg->rel_tol > 0.0) || !(cfg->abs_tol > 0.0))
    return fail(ctx, MPSG_E_ARG, "solver: tolerances must be positive");
  if (cfg->max_iters < 1) return fail(ctx, MPSG_E_ARG, "solver: max_iters must be at least 1");
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "solver: complex matrices are not supported by cg");
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "cg: unknown order %d", order);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  switch (A->K) {
    case 2: return run_dcg<2>(A, order, b_local, x0_local, cfg, x_out_local, history, history_cap, report);
    case 3: return run_dcg<3>(A, order, b_local, x0_local, cfg, x_out_local, history, history_cap, report);
    case 4: return run_dcg<4>(A, order, b_local, x0_local, cfg, x_out_local, history, history_cap, report);
  }
  return fail(ctx, MPSG_E_ARG, "cg: unsupported K");
}

int mpsg_dsolve(mpsg_dcsr* A, int order, const double* b_local, const double* x0_local,
                const mpsg_solver_config* cfg, double* x_out_local, double* history, int64_t history_cap,
                mpsg_cg_report* report) {
  if (!A || !cfg || !report || (!b_local && A->row_end > A->row_begin)) return MPSG_E_ARG;
  mpsg_ctx* ctx = A->comm->ctx;
  // SolverConfig::validate (krylov.hpp:69-75)
  if (!(cfg->rel_tol > 0.0) || !(cfg->abs_tol > 0.0))
    return fail(ctx, MPSG_E_ARG, "solver: tolerances must be positive");
  if (cfg->max_iters < 1) return fail(ctx, MPSG_E_ARG, "solver: max_iters must be at least 1");
  if (cfg->threads < 1) return fail(ctx, MPSG_E_ARG, "solver: threads must be at least 1");
  if (cfg->method < MPSG_CG || cfg->method > MPSG_GPBICG)
    return fail(ctx, MPSG_E_ARG, "solve: unknown method %d", cfg->method);
  if (cfg->dot_order != MPSG_DOT_TREE && cfg->dot_order != MPSG_DOT_SEQUENTIAL)
    return fail(ctx, MPSG_E_ARG, "solve: unknown dot order %d", cfg->dot_order);
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "solver: complex matrices are not supported");
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "solve: unknown order %d", order);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  switch (A->K) {
    case 2: return krylov_driver<2>(ctx, A->local, A, cfg, order, b_local, x0_local, x_out_local, history, history_cap, report);
    case 3: return krylov_driver<3>(ctx, A->local, A, cfg, order, b_local, x0_local, x_out_local, history, history_cap, report);
    case 4: return krylov_driver<4>(ctx, A->local, A, cfg, order, b_local, x0_local, x_out_local, history, history_cap, report);
  }
  return fail(ctx, MPSG_E_ARG, "solve: unsupported K");
}

}  // extern "C"
