// capi.cu -- host side of the C ABI declared in include/mpsg.h.
//
// Owns device memory, streams and the one-time re-layout of a reference CSR
// (int64 indptr/indices + K SoA planes, sparse.hpp:47-78) into the device
// layout described in layout.h, and dispatches the SpMV / CG launchers that
// live in the per-K translation units.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include <unistd.h>

#include "internal.h"

#include <omp.h>

using namespace mpsg;

namespace {

template <class T>
int dev_alloc(mpsg_ctx* ctx, mpsg_csr* A, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
  A->device_bytes += (int64_t)(count * sizeof(T));
  return MPSG_OK;
}

int ensure_scratch(mpsg_ctx* ctx, int slot, size_t bytes) {
  if (ctx->dcap[slot] >= bytes) return MPSG_OK;
  if (ctx->dbuf[slot]) cudaFree(ctx->dbuf[slot]);
  ctx->dbuf[slot] = nullptr;
  ctx->dcap[slot] = 0;
  CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(&ctx->dbuf[slot]), bytes ? bytes : 8));
  ctx->dcap[slot] = bytes;
  return MPSG_OK;
}

// ---- upload helper kernels --------------------------------------------
// SELL build: thread per slot, k loop; padding gets col 0 / value 0.
__global__ void build_sell_kernel(int64_t nslots, int C, const int64_t* slice_ptr,
                                  const int* slot_row, const int* slot_len, const int64_t* indptr,
                                  const int64_t* indices, const double* planes, int nplanes,
                                  int64_t nnz, int64_t ncols, int* scol, double* sval,
                                  int64_t stride, int* bad) {
  int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (slot >= nslots) return;
  const int64_t s = slot / C, t = slot % C;
  const int64_t base = slice_ptr[s] + t;
  const int slen = (int)((slice_ptr[s + 1] - slice_ptr[s]) / C);
  const int row = slot_row[slot], len = slot_len[slot];
  const int64_t src0 = row >= 0 ? indptr[row] : 0;
  for (int k = 0; k < slen; ++k) {
    const int64_t dst = base + (int64_t)k * C;
    if (k < len) {
      const int64_t c = indices[src0 + k];
      if (c < 0 || c >= ncols) *bad = 1;
      scol[dst] = (int)c;
      for (int j = 0; j < nplanes; ++j) sval[j * stride + dst] = planes[j * nnz + src0 + k];
    } else {
      scol[dst] = 0;
      for (int j = 0; j < nplanes; ++j) sval[j * stride + dst] = 0.0;
    }
  }
}

// Long store build: one block per long row, contiguous copy.
__global__ void build_long_kernel(const int* lrow, const int64_t* lptr, const int64_t* indptr,
                                  const int64_t* indices, const double* planes, int nplanes,
                                  int64_t nnz, int64_t ncols, int* lcol, double* lval,
                                  int64_t stride, int* bad) {
  const int r = blockIdx.x;
  const int64_t src0 = indptr[lrow[r]];
  const int64_t dst0 = lptr[r], len = lptr[r + 1] - dst0;
  for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
    const int64_t c = indices[src0 + k];
    if (c < 0 || c >= ncols) *bad = 1;
    lcol[dst0 + k] = (int)c;
    for (int j = 0; j < nplanes; ++j) lval[j * stride + dst0 + k] = planes[j * nnz + src0 + k];
  }
}

__global__ void remap_kernel(int* ids, int64_t n, const int* map) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && ids[i] >= 0) ids[i] = map[ids[i]];
}

void free_csr(mpsg_csr* A) {
  if (!A) return;
  free_csr(A->trans);
  void* ptrs[] = {A->slice_ptr, A->slot_row,    A->slot_len, A->scol,      A->sval,
                  A->lrow,      A->lptr,        A->lcol,     A->lval,      A->chunk_row,
                  A->chunk_beg, A->chunk_end,   A->chunk_slot, A->chunk_first, A->partial,
                  A->counter,   A->xpad};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete A;
}

std::string dim_msg(const char* what, int64_t vsize, int64_t ncols) {
  // kernels.hpp:333-339
  return std::string(what) + ": vector length " + std::to_string(vsize) +
         " does not match matrix dimension " + std::to_string(ncols);
}


}  // namespace

namespace mpsg {
int remap_rows(mpsg_ctx* ctx, mpsg_csr* A, const std::vector<int>& map) {
  int* d_map = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&d_map, std::max<size_t>(map.size(), 1) * sizeof(int)));
  cudaStream_t st = ctx->stream;
  cudaError_t e = cudaMemcpyAsync(d_map, map.data(), map.size() * sizeof(int), cudaMemcpyHostToDevice, st);
  const int64_t nslots = A->nslices * A->C;
  if (e == cudaSuccess && nslots > 0)
    remap_kernel<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(A->slot_row, nslots, d_map);
  if (e == cudaSuccess && A->nlong > 0)
    remap_kernel<<<(unsigned)((A->nlong + 255) / 256), 256, 0, st>>>(A->lrow, A->nlong, d_map);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_map);
  if (e != cudaSuccess) return fail(ctx, MPSG_E_CUDA, "remap_rows: %s", cudaGetErrorString(e));
  A->part_slice.clear();  // host-call output parts index the old rows
  A->part_row.clear();
  return MPSG_OK;
}

// DD / QD device vectors are read and written with 128-bit (and, 32-byte
// aligned, 256-bit) accesses: they must be 16-byte aligned (any cudaMalloc
// pointer, and any element offset into one, is).  TD elements are 24 bytes and
// take 64-bit accesses.
static int check_vec_align(mpsg_ctx* ctx, const mpsg_csr* A, const double* xre, const double* xim,
                           const double* yre, const double* yim) {
  const uintptr_t m = (A->K == 3) ? 7 : 15;
  const uintptr_t all = reinterpret_cast<uintptr_t>(xre) | reinterpret_cast<uintptr_t>(yre) |
                        (A->cplx ? reinterpret_cast<uintptr_t>(xim) | reinterpret_cast<uintptr_t>(yim) : 0);
  if (all & m)
    return mpsg::fail(ctx, MPSG_E_ARG, "spmv: device vectors must be %d-byte aligned for K = %d", (int)m + 1, A->K);
  return MPSG_OK;
}

int launch_spmv(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* xre, const double* xim,
                double* yre, double* yim, cudaStream_t st, bool conj) {
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "spmv: unknown order %d", order);
  if (A->nrows == 0) return MPSG_OK;
  if (int rc = check_vec_align(ctx, A, xre, xim, yre, yim)) return rc;
  if (!A->cplx) {
    switch (A->K) {
      case 2: return launch_spmv_k<2, false>(ctx, A, order, xre, xim, yre, yim, st, conj, -2);
      case 3: return launch_spmv_k<3, false>(ctx, A, order, xre, xim, yre, yim, st, conj, -2);
      case 4: return launch_spmv_k<4, false>(ctx, A, order, xre, xim, yre, yim, st, conj, -2);
    }
  } else {
    switch (A->K) {
      case 2: return launch_spmv_k<2, true>(ctx, A, order, xre, xim, yre, yim, st, conj, -2);
      case 3: return launch_spmv_k<3, true>(ctx, A, order, xre, xim, yre, yim, st, conj, -2);
      case 4: return launch_spmv_k<4, true>(ctx, A, order, xre, xim, yre, yim, st, conj, -2);
    }
  }
  return fail(ctx, MPSG_E_ARG, "spmv: unsupported K %d", A->K);
}

int launch_spmv_part(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* xre, const double* xim,
                     double* yre, double* yim, cudaStream_t st, bool conj, int part) {
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "spmv: unknown order %d", order);
  if (A->nrows == 0) return MPSG_OK;
  if (int rc = check_vec_align(ctx, A, xre, xim, yre, yim)) return rc;
  switch (A->K * 2 + (A->cplx ? 1 : 0)) {
    case 4: return launch_spmv_k<2, false>(ctx, A, order, xre, xim, yre, yim, st, conj, part);
    case 5: return launch_spmv_k<2, true>(ctx, A, order, xre, xim, yre, yim, st, conj, part);
    case 6: return launch_spmv_k<3, false>(ctx, A, order, xre, xim, yre, yim, st, conj, part);
    case 7: return launch_spmv_k<3, true>(ctx, A, order, xre, xim, yre, yim, st, conj, part);
    case 8: return launch_spmv_k<4, false>(ctx, A, order, xre, xim, yre, yim, st, conj, part);
    case 9: return launch_spmv_k<4, true>(ctx, A, order, xre, xim, yre, yim, st, conj, part);
  }
  return fail(ctx, MPSG_E_ARG, "spmv: unsupported K %d", A->K);
}

}  // namespace mpsg

namespace {
// Host-pointer SpMV with the result copy overlapped: x goes up, then the
// long rows and the SELL parts (A->part_slice) run in order on the compute
// stream, each part's rows (A->part_row) going back to the host on the copy
// stream as soon as that part finishes.  ny = 1 (real) or 2 (complex)
// device/host result pairs.
int spmv_host_overlapped(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* dx0, const double* dx1,
                         double* dy0, double* dy1, double* hy0, double* hy1, bool conj) {
  cudaStream_t st = ctx->stream;
  const size_t row_b = (size_t)A->K * sizeof(double);
  const int P = (int)A->part_slice.size() - 1;
  int rc;
  if ((rc = launch_spmv_part(ctx, A, order, dx0, dx1, dy0, dy1, st, conj, -1))) return rc;
  for (int p = 0; p < P; ++p) {
    if ((rc = launch_spmv_part(ctx, A, order, dx0, dx1, dy0, dy1, st, conj, p))) return rc;
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_part[p], st));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy, ctx->ev_part[p], 0));
    const int64_t r0 = A->part_row[(size_t)p], r1 = A->part_row[(size_t)p + 1];
    if (r1 > r0) {
      CUDA_TRY(ctx, cudaMemcpyAsync(hy0 + r0 * A->K, dy0 + r0 * A->K, (size_t)(r1 - r0) * row_b,
                                    cudaMemcpyDeviceToHost, ctx->copy));
      if (hy1)
        CUDA_TRY(ctx, cudaMemcpyAsync(hy1 + r0 * A->K, dy1 + r0 * A->K, (size_t)(r1 - r0) * row_b,
                                      cudaMemcpyDeviceToHost, ctx->copy));
    }
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->copy));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MPSG_OK;
}
// ---- pageable host vectors ---------------------------------------------
// A std::vector / numpy array is pageable: the driver's own staging copies run
// at ~16 GB/s.  Instead: 8 MB chunks through two pinned slots, the host-side
// copy into / out of a slot done by OpenMP threads while the other slot's DMA
// runs (MPSG_STAGE_HOST=0 falls back to the driver).
constexpr size_t HCHUNK = 8u << 20;
bool host_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}
int ensure_hslots(mpsg_ctx* ctx) {
  if (ctx->hslot_cap >= HCHUNK) return MPSG_OK;
  for (int i = 0; i < 2; ++i) {
    CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->hslot[i]), HCHUNK, cudaHostAllocDefault));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->hslot_ev[i], cudaEventDisableTiming));
  }
  ctx->hslot_cap = HCHUNK;
  return MPSG_OK;
}
void par_copy(void* dst, const void* src, size_t n) {
  const int T = (int)std::min<size_t>(8, std::max<size_t>(1, n >> 20));  // >= 1 MB per thread
#pragma omp parallel for num_threads(T) schedule(static)
  for (int t = 0; t < T; ++t) {
    const size_t a = n * (size_t)t / (size_t)T, b = n * (size_t)(t + 1) / (size_t)T;
    std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  }
}
int h2d_staged(mpsg_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  size_t i = 0;
  for (size_t off = 0; off < bytes; off += HCHUNK, ++i) {
    const int sl = (int)(i & 1);
    const size_t len = std::min(HCHUNK, bytes - off);
    if (i >= 2) CUDA_TRY(ctx, cudaEventSynchronize(ctx->hslot_ev[sl]));
    par_copy(ctx->hslot[sl], static_cast<const char*>(src) + off, len);
    CUDA_TRY(ctx, cudaMemcpyAsync(static_cast<char*>(dst) + off, ctx->hslot[sl], len, cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->hslot_ev[sl], st));
  }
  return MPSG_OK;
}
int d2h_staged(mpsg_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  int psl = -1;
  size_t poff = 0, plen = 0, i = 0;
  for (size_t off = 0; off < bytes; off += HCHUNK, ++i) {
    const int sl = (int)(i & 1);
    const size_t len = std::min(HCHUNK, bytes - off);
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->hslot[sl], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                                  st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->hslot_ev[sl], st));
    if (psl >= 0) {  // the previous chunk drains while this one crosses PCIe
      CUDA_TRY(ctx, cudaEventSynchronize(ctx->hslot_ev[psl]));
      par_copy(static_cast<char*>(dst) + poff, ctx->hslot[psl], plen);
    }
    psl = sl;
    poff = off;
    plen = len;
  }
  if (psl >= 0) {
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->hslot_ev[psl]));
    par_copy(static_cast<char*>(dst) + poff, ctx->hslot[psl], plen);
  }
  return MPSG_OK;
}

bool can_overlap(const mpsg_ctx* ctx, const mpsg_csr* A) {
  return ctx->overlap && ctx->copy && A->part_slice.size() >= 3 && A->part_slice.size() <= 17;
}
}  // namespace

namespace {
// Text of the last failed mpsg_ctx_create on this host thread (there is no
// context to hang it on); read with mpsg_create_error().
thread_local std::string g_create_err;

cudaError_t ctx_init(mpsg_ctx* ctx, int device) {
  cudaError_t e = cudaSetDevice(device);
  // cudaSetDevice is lazy: force primary-context creation here so a busy or
  // unusable device is reported by this call, not by the first launch
  if (e == cudaSuccess) e = cudaFree(nullptr);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_side0, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_side1, cudaEventDisableTiming);
  for (auto& ev : ctx->ev_part)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  return e;
}
}  // namespace

// ==========================================================================
extern "C" {

const char* mpsg_version(void) { return "mpsg 0.1 (sm_100a)"; }

const char* mpsg_create_error(void) { return g_create_err.c_str(); }

// The one retry policy of the library (the C++ Context, the Python Context and
// the CLI all come through here): a device that is momentarily held by another
// process (cudaErrorDevicesUnavailable -- an exclusive-process GPU whose
// previous owner is still tearing its context down) is retried for up to ~2 s;
// every other error fails at once.  On failure everything created so far is
// released and the CUDA error text is kept for mpsg_create_error().
int mpsg_ctx_create(int device, mpsg_ctx** out) {
  if (!out) return MPSG_E_ARG;
  *out = nullptr;
  g_create_err.clear();
  mpsg_ctx* ctx = nullptr;
  cudaError_t e = cudaSuccess;
  for (int attempt = 0;; ++attempt) {
    ctx = new mpsg_ctx();
    ctx->device = device;
    e = ctx_init(ctx, device);
    if (e == cudaSuccess) break;
    mpsg_ctx_destroy(ctx);
    ctx = nullptr;
    cudaGetLastError();
    if (e != cudaErrorDevicesUnavailable || attempt >= 8) break;
    usleep(250000);
  }
  if (!ctx) {
    g_create_err = std::string("mpsg_ctx_create(device=") + std::to_string(device) + "): " +
                   cudaGetErrorName(e) + ": " + cudaGetErrorString(e);
    return MPSG_E_CUDA;
  }
  ctx->stream = ctx->own_stream;
  {
    // persisting L2 set-aside for the gathered vector (see launch_win).  Off
    // by default: measured slower on B200 for every config (profiles/
    // r01b_l2_persist.txt); MPSG_L2_PERSIST=1 turns it on.
    const char* env = std::getenv("MPSG_L2_PERSIST");
    int maxp = 0;
    if (env && env[0] == '1' &&
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device) == cudaSuccess && maxp > 0 &&
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp) == cudaSuccess)
      ctx->persist_max = (size_t)maxp;
    cudaGetLastError();
  }
  if (const char* s = std::getenv("MPSG_LONG_THRESHOLD")) ctx->long_threshold = std::atoll(s);
  if (const char* s = std::getenv("MPSG_SIGMA")) ctx->sigma = std::atoll(s);
  if (const char* s = std::getenv("MPSG_FAST_CHUNK")) ctx->fast_chunk = std::atoll(s);
  if (const char* s = std::getenv("MPSG_COLBLOCK_BYTES")) ctx->colblock_bytes = std::atoll(s);
  if (const char* s = std::getenv("MPSG_OVERLAP")) ctx->overlap = s[0] != '0';
  if (const char* s = std::getenv("MPSG_STAGE_HOST")) ctx->stage_host = s[0] != '0';
  if (const char* s = std::getenv("MPSG_COLBLOCK_MIN")) ctx->colblock_min = std::atoll(s);
  *out = ctx;
  return MPSG_OK;
}

void mpsg_ctx_destroy(mpsg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (auto& p : ctx->dbuf)
    if (p) cudaFree(p);
  for (int i = 0; i < 2; ++i) {
    if (ctx->hslot[i]) cudaFreeHost(ctx->hslot[i]);
    if (ctx->hslot_ev[i]) cudaEventDestroy(ctx->hslot_ev[i]);
  }
  if (ctx->seg_bounds) cudaFree(ctx->seg_bounds);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  for (auto& ev : ctx->ev_part)
    if (ev) cudaEventDestroy(ev);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_side0) cudaEventDestroy(ctx->ev_side0);
  if (ctx->ev_side1) cudaEventDestroy(ctx->ev_side1);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* mpsg_last_error(const mpsg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int mpsg_ctx_set_stream(mpsg_ctx* ctx, void* stream) {
  if (!ctx) return MPSG_E_ARG;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return MPSG_OK;
}

int mpsg_ctx_set_layout(mpsg_ctx* ctx, int64_t long_threshold, int64_t sigma, int64_t fast_chunk) {
  if (!ctx) return MPSG_E_ARG;
  if (long_threshold > 0) ctx->long_threshold = long_threshold;
  if (sigma > 0) ctx->sigma = sigma;
  if (fast_chunk > 0) {
    if (fast_chunk % 32) return fail(ctx, MPSG_E_ARG, "fast_chunk must be a multiple of 32");
    ctx->fast_chunk = fast_chunk;
  }
  return MPSG_OK;
}

int mpsg_ctx_synchronize(mpsg_ctx* ctx) {
  if (!ctx) return MPSG_E_ARG;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return MPSG_OK;
}

int mpsg_csr_upload(mpsg_ctx* ctx, int K, int is_complex, int64_t nrows, int64_t ncols,
                    const int64_t* indptr, const int64_t* indices, const double* const* planes,
                    mpsg_csr** out) {
  return mpsg_csr_upload_ex(ctx, K, is_complex ? MPSG_CSR_COMPLEX : 0, nrows, ncols, indptr, indices, planes, out);
}

int mpsg_csr_upload_ex(mpsg_ctx* ctx, int K, int flags, int64_t nrows, int64_t ncols, const int64_t* indptr,
                       const int64_t* indices, const double* const* planes, mpsg_csr** out) {
  if (!ctx || !out) return MPSG_E_ARG;
  *out = nullptr;
  const int is_complex = (flags & MPSG_CSR_COMPLEX) != 0;
  const bool mixed = (flags & MPSG_CSR_MIXED) != 0;
  if (K < 2 || K > 4) return fail(ctx, MPSG_E_ARG, "csr_upload: K must be 2, 3 or 4 (got %d)", K);
  if (flags & ~(MPSG_CSR_COMPLEX | MPSG_CSR_MIXED | MPSG_CSR_TRANSPOSE))
    return fail(ctx, MPSG_E_ARG, "csr_upload: unknown flags 0x%x", flags);
  if (nrows < 0 || ncols < 0 || !indptr) return fail(ctx, MPSG_E_ARG, "csr_upload: bad shape");
  const int64_t I32 = std::numeric_limits<int>::max();
  if (nrows > I32 || ncols > I32)
    return fail(ctx, MPSG_E_RANGE, "csr_upload: %lld x %lld exceeds the int32 index range",
                (long long)nrows, (long long)ncols);
  if (indptr[0] != 0) return fail(ctx, MPSG_E_STRUCT, "csr_upload: indptr[0] must be 0");
  const int64_t nnz = indptr[nrows];
  const int nplanes = (mixed ? 1 : K) * (is_complex ? 2 : 1);
  if (nnz > 0 && (!indices || !planes)) return fail(ctx, MPSG_E_ARG, "csr_upload: null arrays");
  for (int j = 0; j < nplanes && nnz > 0; ++j)
    if (!planes[j]) return fail(ctx, MPSG_E_ARG, "csr_upload: null plane %d", j);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;

  auto* A = new mpsg_csr();
  std::unique_ptr<mpsg_csr, void (*)(mpsg_csr*)> holder(A, free_csr);
  A->K = K;
  A->cplx = is_complex != 0;
  A->mixed = mixed;
  A->nrows = nrows;
  A->ncols = ncols;
  A->nnz = nnz;
  A->C = A->cplx ? 16 : 32;
  A->chunk = ctx->fast_chunk;
  const int C = A->C;
  const int64_t T = ctx->long_threshold;

  // ---- host planning: row classes, windowed length sort, slices
  std::vector<int> short_rows;
  std::vector<int> long_rows;
  short_rows.reserve((size_t)nrows);
  for (int64_t i = 0; i < nrows; ++i) {
    const int64_t len = indptr[i + 1] - indptr[i];
    if (len < 0) return fail(ctx, MPSG_E_STRUCT, "csr_upload: indptr not monotone at row %lld", (long long)i);
    if (len > T)
      long_rows.push_back((int)i);
    else
      short_rows.push_back((int)i);
  }
  // Long rows longest first: the exact orders run one serial chain (four with
  // lanes on) per row, so the kernel ends when its longest row does -- a
  // 50000-element row scheduled last would add its whole chain to the tail.
  std::stable_sort(long_rows.begin(), long_rows.end(), [&](int a, int b) {
    return indptr[a + 1] - indptr[a] > indptr[b + 1] - indptr[b];
  });
  // Output parts for the host-pointer calls: consecutive sort windows write a
  // contiguous range of y rows (plus long rows, computed first), so the
  // device->host copy of part p overlaps the SELL launch of part p+1.
  {
    const int64_t W = std::max<int64_t>(1, ctx->sigma);
    const int64_t nwin = ((int64_t)short_rows.size() + W - 1) / W;
    // P equal parts (env MPSG_PARTS): each part is its own SELL launch, whose
    // tail costs more than the shorter copy-engine wait of finer parts saves
    // (config 2 QD end to end: 2 / 4 / 8 / 12 / 16 parts = 22.3 / 23.6 / 21.9 /
    // 20.3 / 17.9 Gnnz/s; geometric sizes were worse, profiles/r01b_variants.txt).
    const char* ep = std::getenv("MPSG_PARTS");
    const int64_t P = std::min<int64_t>(ep ? std::max(2, std::min(16, std::atoi(ep))) : 4, nwin);
    if (P >= 2 && W % C == 0) {
      for (int64_t p = 0; p <= P; ++p) {
        const int64_t w = nwin * p / P;
        A->part_slice.push_back(std::min<int64_t>(w * (W / C), ((int64_t)short_rows.size() + C - 1) / C));
        A->part_row.push_back(p == 0 ? 0
                                     : ((p == P || w * W >= (int64_t)short_rows.size()) ? nrows
                                                                                       : short_rows[(size_t)(w * W)]));
      }
    }
  }
  // stable counting sort by length, descending, inside windows of sigma rows
  {
    std::vector<int> sorted(short_rows.size());
    std::vector<int64_t> cnt((size_t)T + 2);
    const size_t W = (size_t)std::max<int64_t>(1, ctx->sigma);
    for (size_t w0 = 0; w0 < short_rows.size(); w0 += W) {
      const size_t w1 = std::min(short_rows.size(), w0 + W);
      std::fill(cnt.begin(), cnt.end(), 0);
      for (size_t i = w0; i < w1; ++i) {
        const int64_t len = indptr[short_rows[i] + 1] - indptr[short_rows[i]];
        cnt[(size_t)(T - len)]++;
      }
      int64_t acc = (int64_t)w0;
      for (auto& c : cnt) {
        const int64_t v = c;
        c = acc;
        acc += v;
      }
      for (size_t i = w0; i < w1; ++i) {
        const int64_t len = indptr[short_rows[i] + 1] - indptr[short_rows[i]];
        sorted[(size_t)cnt[(size_t)(T - len)]++] = short_rows[i];
      }
    }
    short_rows.swap(sorted);
  }
  A->nslices = ((int64_t)short_rows.size() + C - 1) / C;
  std::vector<int> slot_row((size_t)(A->nslices * C), -1), slot_len((size_t)(A->nslices * C), 0);
  std::vector<int64_t> slice_ptr((size_t)A->nslices + 1, 0);
  for (int64_t s = 0; s < A->nslices; ++s) {
    int mx = 0;
    for (int t = 0; t < C; ++t) {
      const int64_t i = s * C + t;
      if (i < (int64_t)short_rows.size()) {
        const int row = short_rows[(size_t)i];
        const int len = (int)(indptr[row + 1] - indptr[row]);
        slot_row[(size_t)i] = row;
        slot_len[(size_t)i] = len;
        mx = std::max(mx, len);
      }
    }
    slice_ptr[(size_t)s + 1] = slice_ptr[(size_t)s] + (int64_t)mx * C;
  }
  A->sell_elems = slice_ptr.back();
  // long store plan
  A->nlong = (int64_t)long_rows.size();
  std::vector<int64_t> lptr((size_t)A->nlong + 1, 0);
  for (int64_t r = 0; r < A->nlong; ++r) {
    const int row = long_rows[(size_t)r];
    lptr[(size_t)r + 1] = lptr[(size_t)r] + (indptr[row + 1] - indptr[row]);
  }
  // Fast-order chunks of the long rows.  Each row is cut where its (sorted)
  // columns cross a column-block boundary -- a block = colblock_bytes of x --
  // and every piece into chunks of at most `chunk` elements.  Chunks are then
  // ordered block-major, so the warps running at any one time gather from
  // one block of x (L2-resident) instead of all of it.  Slots (the partial
  // sums' combine order) follow row position, so the result does not depend
  // on the blocking.
  std::vector<int> chunk_first((size_t)A->nlong + 1, 0), chunk_row, chunk_slot;
  std::vector<int64_t> chunk_beg, chunk_end;
  {
    const int64_t xb = (int64_t)K * 8 * (A->cplx ? 2 : 1);
    const int64_t W = ctx->colblock_bytes > 0 ? std::max<int64_t>(1, ctx->colblock_bytes / xb) : ncols + 1;
    const int64_t B = std::max<int64_t>(1, (ncols + W - 1) / W);
    std::vector<std::vector<std::array<int64_t, 4>>> per_block((size_t)B);  // (row, beg, end, slot)
    int slot = 0;
    for (int64_t r = 0; r < A->nlong; ++r) {
      const int row = long_rows[(size_t)r];
      const int64_t src = indptr[row], len = indptr[row + 1] - src;
      bool sorted = true;
      if (B > 1 && len >= ctx->colblock_min)
        for (int64_t k = 1; k < len && sorted; ++k) sorted = indices[src + k] >= indices[src + k - 1];
      const bool split = B > 1 && len >= ctx->colblock_min && sorted;
      int64_t k = 0;
      while (k < len) {
        const int64_t blk = split ? std::min<int64_t>(B - 1, indices[src + k] / W) : 0;
        int64_t kend = len;
        if (split && blk + 1 < B) {  // first position with column >= (blk+1)*W
          kend = std::lower_bound(indices + src + k, indices + src + len, (blk + 1) * W) - (indices + src);
        }
        for (int64_t c = k; c < kend; c += A->chunk)
          per_block[(size_t)blk].push_back({r, lptr[(size_t)r] + c, lptr[(size_t)r] + std::min(kend, c + A->chunk),
                                            (int64_t)slot++});
        k = kend;
      }
      chunk_first[(size_t)r + 1] = slot;
    }
    for (auto& v : per_block)
      for (auto& c : v) {
        chunk_row.push_back((int)c[0]);
        chunk_beg.push_back(c[1]);
        chunk_end.push_back(c[2]);
        chunk_slot.push_back((int)c[3]);
      }
  }
  A->long_nnz = lptr.back();
  A->nchunks = (int64_t)chunk_row.size();

  // ---- device staging of the reference arrays
  int64_t* d_indptr = nullptr;
  int64_t* d_indices = nullptr;
  double* d_planes = nullptr;
  int* d_bad = nullptr;
  auto free_stage = [&]() {
    if (d_indptr) cudaFree(d_indptr);
    if (d_indices) cudaFree(d_indices);
    if (d_planes) cudaFree(d_planes);
    if (d_bad) cudaFree(d_bad);
  };
  struct StageGuard {
    std::function<void()> f;
    ~StageGuard() { f(); }
  };
  StageGuard sg{free_stage};
  CUDA_TRY(ctx, cudaMalloc(&d_indptr, (size_t)(nrows + 1) * sizeof(int64_t)));
  CUDA_TRY(ctx, cudaMalloc(&d_indices, (size_t)std::max<int64_t>(nnz, 1) * sizeof(int64_t)));
  CUDA_TRY(ctx, cudaMalloc(&d_planes, (size_t)std::max<int64_t>(nnz, 1) * nplanes * sizeof(double)));
  CUDA_TRY(ctx, cudaMalloc(&d_bad, sizeof(int)));
  CUDA_TRY(ctx, cudaMemsetAsync(d_bad, 0, sizeof(int), st));
  CUDA_TRY(ctx, cudaMemcpyAsync(d_indptr, indptr, (size_t)(nrows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  if (nnz > 0) {
    CUDA_TRY(ctx, cudaMemcpyAsync(d_indices, indices, (size_t)nnz * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    for (int j = 0; j < nplanes; ++j)
      CUDA_TRY(ctx, cudaMemcpyAsync(d_planes + (size_t)j * nnz, planes[j], (size_t)nnz * sizeof(double),
                                    cudaMemcpyHostToDevice, st));
  }
  int rc;
  // SELL store
  if ((rc = dev_alloc(ctx, A, &A->slice_ptr, (size_t)A->nslices + 1))) return rc;
  if ((rc = dev_alloc(ctx, A, &A->slot_row, (size_t)(A->nslices * C)))) return rc;
  if ((rc = dev_alloc(ctx, A, &A->slot_len, (size_t)(A->nslices * C)))) return rc;
  if ((rc = dev_alloc(ctx, A, &A->scol, (size_t)A->sell_elems))) return rc;
  if ((rc = dev_alloc(ctx, A, &A->sval, (size_t)A->sell_elems * nplanes))) return rc;
  CUDA_TRY(ctx, cudaMemcpyAsync(A->slice_ptr, slice_ptr.data(), slice_ptr.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  if (A->nslices) {
    CUDA_TRY(ctx, cudaMemcpyAsync(A->slot_row, slot_row.data(), slot_row.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(A->slot_len, slot_len.data(), slot_len.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    const int64_t nslots = A->nslices * C;
    build_sell_kernel<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(
        nslots, C, A->slice_ptr, A->slot_row, A->slot_len, d_indptr, d_indices, d_planes, nplanes, nnz,
        ncols, A->scol, A->sval, A->sell_elems, d_bad);
    CUDA_TRY(ctx, cudaGetLastError());
  }
  // TD x padded to 32 bytes per element for the FAST short-row kernel (one
  // 256-bit gather instead of three 64-bit ones: cfg2 TD 252 -> 224 us).  The
  // re-layout costs a pass over x (56 bytes per column) per SpMV, so only
  // matrices with enough gathers per column take it (cfg5, 7 per column:
  // 106 -> 132 us with it).
  if (K == 3 && !A->cplx && !A->mixed && (nnz - A->long_nnz) >= 12 * ncols && nnz >= (1 << 20))
    if ((rc = dev_alloc(ctx, A, &A->xpad, (size_t)ncols * 4))) return rc;
  // long store
  if (A->nlong) {
    const int NS = A->cplx ? 4 : 1;
    if ((rc = dev_alloc(ctx, A, &A->lrow, (size_t)A->nlong))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->lptr, (size_t)A->nlong + 1))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->lcol, (size_t)A->long_nnz))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->lval, (size_t)A->long_nnz * nplanes))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->chunk_row, (size_t)A->nchunks))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->chunk_beg, (size_t)A->nchunks))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->chunk_end, (size_t)A->nchunks))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->chunk_slot, (size_t)A->nchunks))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->chunk_first, (size_t)A->nlong + 1))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->partial, (size_t)A->nchunks * NS * K))) return rc;
    if ((rc = dev_alloc(ctx, A, &A->counter, (size_t)A->nlong))) return rc;
    CUDA_TRY(ctx, cudaMemcpyAsync(A->lrow, long_rows.data(), long_rows.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(A->lptr, lptr.data(), lptr.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(A->chunk_row, chunk_row.data(), chunk_row.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(A->chunk_beg, chunk_beg.data(), chunk_beg.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(A->chunk_end, chunk_end.data(), chunk_end.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(A->chunk_slot, chunk_slot.data(), chunk_slot.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(A->chunk_first, chunk_first.data(), chunk_first.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemsetAsync(A->counter, 0, (size_t)A->nlong * sizeof(unsigned), st));
    build_long_kernel<<<(unsigned)A->nlong, 256, 0, st>>>(A->lrow, A->lptr, d_indptr, d_indices, d_planes,
                                                          nplanes, nnz, ncols, A->lcol, A->lval,
                                                          A->long_nnz, d_bad);
    CUDA_TRY(ctx, cudaGetLastError());
  }
  int bad = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (bad) return fail(ctx, MPSG_E_RANGE, "csr_upload: column index outside [0, %lld)", (long long)ncols);
  if (flags & MPSG_CSR_TRANSPOSE) {
    A->host_indptr.assign(indptr, indptr + nrows + 1);
    // A^T on the host (stable counting sort by column, as transpose_csr,
    // sparse.hpp:139-163: the rows of A^T list their entries in ascending
    // original row), uploaded as its own device matrix.  Row j of A^T summed
    // in row order is exactly the reference sptmv's accumulation into y[j]
    // at one thread (kernels.hpp:212-225): acc_j += A_ij v_i, i ascending.
    std::vector<int64_t> tptr((size_t)ncols + 1, 0), tidx((size_t)nnz);
    std::vector<double> tval((size_t)nnz * nplanes);
    for (int64_t k = 0; k < nnz; ++k) tptr[(size_t)indices[k] + 1]++;
    for (int64_t j = 0; j < ncols; ++j) tptr[(size_t)j + 1] += tptr[(size_t)j];
    std::vector<int64_t> pos(tptr.begin(), tptr.end() - 1);
    for (int64_t i = 0; i < nrows; ++i)
      for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
        const int64_t d = pos[(size_t)indices[k]]++;
        tidx[(size_t)d] = i;
        for (int j = 0; j < nplanes; ++j) tval[(size_t)j * nnz + d] = planes[j][k];
      }
    std::vector<const double*> tpl((size_t)nplanes);
    for (int j = 0; j < nplanes; ++j) tpl[(size_t)j] = tval.data() + (size_t)j * nnz;
    int rct = mpsg_csr_upload_ex(ctx, K, flags & ~MPSG_CSR_TRANSPOSE, ncols, nrows, tptr.data(), tidx.data(),
                                 tpl.data(), &A->trans);
    if (rct) return rct;
  }
  *out = holder.release();
  return MPSG_OK;
}

void mpsg_csr_destroy(mpsg_csr* A) { free_csr(A); }

int mpsg_csr_get_stats(const mpsg_csr* A, mpsg_csr_stats* o) {
  if (!A || !o) return MPSG_E_ARG;
  o->nrows = A->nrows;
  o->ncols = A->ncols;
  o->nnz = A->nnz;
  o->K = A->K;
  o->is_complex = A->cplx;
  o->nslices = A->nslices;
  o->sell_elems = A->sell_elems;
  o->nlong = A->nlong;
  o->long_nnz = A->long_nnz;
  o->nchunks = A->nchunks;
  o->device_bytes = A->device_bytes + (A->trans ? A->trans->device_bytes : 0);
  o->is_mixed = A->mixed;
  o->has_transpose = A->trans != nullptr;
  return MPSG_OK;
}

int mpsg_spmv_dev(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* d_x, double* d_y,
                  void* stream) {
  if (!ctx || !A) return MPSG_E_ARG;
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "spmv: matrix is complex, use mpsg_spmv_complex");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return launch_spmv(ctx, A, order, d_x, nullptr, d_y, nullptr, st);
}

int mpsg_spmv(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t xlen, const double* x,
              double* y) {
  if (!ctx || !A) return MPSG_E_ARG;
  if (xlen != A->ncols) return fail(ctx, MPSG_E_DIM, "%s", dim_msg("spmv", xlen, A->ncols).c_str());
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "spmv: matrix is complex, use mpsg_spmv_complex");
  const size_t xb = (size_t)A->ncols * A->K * sizeof(double), yb = (size_t)A->nrows * A->K * sizeof(double);
  int rc;
  if ((rc = ensure_scratch(ctx, 0, xb))) return rc;
  if ((rc = ensure_scratch(ctx, 1, yb))) return rc;
  cudaStream_t st = ctx->stream;
  const bool px = xb && host_pageable(x), py = yb && host_pageable(y);
  if (ctx->stage_host && (px || py) && ensure_hslots(ctx) == MPSG_OK) {
    // pageable vectors: chunked pinned staging both ways
    if (px)
      rc = h2d_staged(ctx, ctx->dbuf[0], x, xb, st);
    else if (xb)
      rc = cudaMemcpyAsync(ctx->dbuf[0], x, xb, cudaMemcpyHostToDevice, st) == cudaSuccess
               ? MPSG_OK
               : fail(ctx, MPSG_E_CUDA, "spmv: x copy failed");
    if (rc) return rc;
    if ((rc = launch_spmv(ctx, A, order, ctx->dbuf[0], nullptr, ctx->dbuf[1], nullptr, st))) return rc;
    if (py)
      rc = d2h_staged(ctx, y, ctx->dbuf[1], yb, st);
    else if (yb)
      rc = cudaMemcpyAsync(y, ctx->dbuf[1], yb, cudaMemcpyDeviceToHost, st) == cudaSuccess
               ? MPSG_OK
               : fail(ctx, MPSG_E_CUDA, "spmv: y copy failed");
    if (rc) return rc;
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    return MPSG_OK;
  }
  if (xb) CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dbuf[0], x, xb, cudaMemcpyHostToDevice, st));
  if (can_overlap(ctx, A))
    return spmv_host_overlapped(ctx, A, order, ctx->dbuf[0], nullptr, ctx->dbuf[1], nullptr, y, nullptr, false);
  if ((rc = launch_spmv(ctx, A, order, ctx->dbuf[0], nullptr, ctx->dbuf[1], nullptr, st))) return rc;
  if (yb) CUDA_TRY(ctx, cudaMemcpyAsync(y, ctx->dbuf[1], yb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MPSG_OK;
}

int mpsg_spmv_complex_dev(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* d_x_re,
                          const double* d_x_im, double* d_y_re, double* d_y_im, void* stream) {
  if (!ctx || !A) return MPSG_E_ARG;
  if (!A->cplx) return fail(ctx, MPSG_E_ARG, "spmv_complex: matrix is real");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return launch_spmv(ctx, A, order, d_x_re, d_x_im, d_y_re, d_y_im, st);
}

int mpsg_spmv_complex(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t xlen,
                      const double* x_re, const double* x_im, double* y_re, double* y_im) {
  if (!ctx || !A) return MPSG_E_ARG;
  if (!A->cplx) return fail(ctx, MPSG_E_ARG, "spmv_complex: matrix is real");
  if (xlen != A->ncols) return fail(ctx, MPSG_E_DIM, "%s", dim_msg("spmv", xlen, A->ncols).c_str());
  const size_t xb = (size_t)A->ncols * A->K * sizeof(double), yb = (size_t)A->nrows * A->K * sizeof(double);
  int rc;
  for (int s = 0; s < 4; ++s)
    if ((rc = ensure_scratch(ctx, s, s < 2 ? xb : yb))) return rc;
  cudaStream_t st = ctx->stream;
  if (xb) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dbuf[0], x_re, xb, cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dbuf[1], x_im, xb, cudaMemcpyHostToDevice, st));
  }
  if (can_overlap(ctx, A))
    return spmv_host_overlapped(ctx, A, order, ctx->dbuf[0], ctx->dbuf[1], ctx->dbuf[2], ctx->dbuf[3], y_re, y_im,
                                false);
  if ((rc = launch_spmv(ctx, A, order, ctx->dbuf[0], ctx->dbuf[1], ctx->dbuf[2], ctx->dbuf[3], st))) return rc;
  if (yb) {
    CUDA_TRY(ctx, cudaMemcpyAsync(y_re, ctx->dbuf[2], yb, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(y_im, ctx->dbuf[3], yb, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MPSG_OK;
}

// ---- transposed products ----------------------------------------------
namespace {
int trans_of(mpsg_ctx* ctx, const mpsg_csr* A, const mpsg_csr** T) {
  if (!A->trans)
    return fail(ctx, MPSG_E_ARG, "sptmv: matrix was uploaded without MPSG_CSR_TRANSPOSE");
  *T = A->trans;
  return MPSG_OK;
}
// Exact orders: the reference sptmv at one thread accumulates y[j] over i
// ascending whether lanes are on or off (SptRow lanes are per-element exact,
// kernels.hpp:227-322), i.e. the lanes-off row sum of A^T.
int torder(int order) { return order == MPSG_ORDER_FAST ? MPSG_ORDER_FAST : MPSG_ORDER_SCALAR; }
}  // namespace

int mpsg_sptmv_dev(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* d_v, double* d_y, void* stream) {
  if (!ctx || !A) return MPSG_E_ARG;
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "sptmv: matrix is complex, use mpsg_sptmv_complex");
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "sptmv: unknown order %d", order);
  const mpsg_csr* T;
  int rc = trans_of(ctx, A, &T);
  if (rc) return rc;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return launch_spmv(ctx, T, torder(order), d_v, nullptr, d_y, nullptr, st);
}

}  // extern "C"

namespace {
// Clears the segment bounds set for one transposed launch.
struct SegScope {
  mpsg_ctx* ctx;
  ~SegScope() { ctx->seg_T = 1; }
};
}  // namespace

int mpsg::set_segments(mpsg_ctx* ctx, const mpsg_csr* A, int order, int threads) {
  ctx->seg_T = 1;
  if (threads <= 1 || order == MPSG_ORDER_FAST || A->nrows == 0) return MPSG_OK;
  ctx->seg_host.assign((size_t)threads + 1, 0);
  mpsg_partition_rows(A->host_indptr.data(), A->nrows, threads, ctx->seg_host.data());
  const size_t b = ctx->seg_host.size() * sizeof(int64_t);
  if (ctx->seg_cap < b) {
    if (ctx->seg_bounds) cudaFree(ctx->seg_bounds);
    ctx->seg_bounds = nullptr;
    ctx->seg_cap = 0;
    CUDA_TRY(ctx, cudaMalloc(&ctx->seg_bounds, b));
    ctx->seg_cap = b;
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->seg_bounds, ctx->seg_host.data(), b, cudaMemcpyHostToDevice, ctx->stream));
  ctx->seg_T = threads;
  return MPSG_OK;
}

extern "C" {

int mpsg_sptmv(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t vlen, const double* v, double* y) {
  return mpsg_sptmv_ex(ctx, A, order, 1, vlen, v, y);
}

int mpsg_sptmv_ex(mpsg_ctx* ctx, const mpsg_csr* A, int order, int threads, int64_t vlen, const double* v,
                  double* y) {
  if (!ctx || !A) return MPSG_E_ARG;
  if (vlen != A->nrows) return fail(ctx, MPSG_E_DIM, "%s", dim_msg("sptmv", vlen, A->nrows).c_str());
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "sptmv: matrix is complex, use mpsg_sptmv_complex");
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "sptmv: unknown order %d", order);
  const mpsg_csr* T;
  int rc = trans_of(ctx, A, &T);
  if (rc) return rc;
  const size_t vb = (size_t)A->nrows * A->K * sizeof(double), yb = (size_t)A->ncols * A->K * sizeof(double);
  if ((rc = ensure_scratch(ctx, 0, vb))) return rc;
  if ((rc = ensure_scratch(ctx, 1, yb))) return rc;
  cudaStream_t st = ctx->stream;
  if (vb) CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dbuf[0], v, vb, cudaMemcpyHostToDevice, st));
  if (yb && T->nnz == 0) CUDA_TRY(ctx, cudaMemsetAsync(ctx->dbuf[1], 0, yb, st));
  SegScope scope{ctx};
  if ((rc = set_segments(ctx, A, order, threads))) return rc;
  if ((rc = launch_spmv(ctx, T, torder(order), ctx->dbuf[0], nullptr, ctx->dbuf[1], nullptr, st))) return rc;
  if (yb) CUDA_TRY(ctx, cudaMemcpyAsync(y, ctx->dbuf[1], yb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MPSG_OK;
}

int mpsg_sptmv_complex_dev(mpsg_ctx* ctx, const mpsg_csr* A, int order, int conjugate, const double* d_v_re,
                           const double* d_v_im, double* d_y_re, double* d_y_im, void* stream) {
  if (!ctx || !A) return MPSG_E_ARG;
  if (!A->cplx) return fail(ctx, MPSG_E_ARG, "sptmv_complex: matrix is real");
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "sptmv: unknown order %d", order);
  const mpsg_csr* T;
  int rc = trans_of(ctx, A, &T);
  if (rc) return rc;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return launch_spmv(ctx, T, torder(order), d_v_re, d_v_im, d_y_re, d_y_im, st, conjugate != 0);
}

int mpsg_sptmv_complex(mpsg_ctx* ctx, const mpsg_csr* A, int order, int conjugate, int64_t vlen,
                       const double* v_re, const double* v_im, double* y_re, double* y_im) {
  return mpsg_sptmv_complex_ex(ctx, A, order, 1, conjugate, vlen, v_re, v_im, y_re, y_im);
}

int mpsg_sptmv_complex_ex(mpsg_ctx* ctx, const mpsg_csr* A, int order, int threads, int conjugate, int64_t vlen,
                          const double* v_re, const double* v_im, double* y_re, double* y_im) {
  if (!ctx || !A) return MPSG_E_ARG;
  if (!A->cplx) return fail(ctx, MPSG_E_ARG, "sptmv_complex: matrix is real");
  if (vlen != A->nrows) return fail(ctx, MPSG_E_DIM, "%s", dim_msg("sptmv", vlen, A->nrows).c_str());
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "sptmv: unknown order %d", order);
  const mpsg_csr* T;
  int rc = trans_of(ctx, A, &T);
  if (rc) return rc;
  const size_t vb = (size_t)A->nrows * A->K * sizeof(double), yb = (size_t)A->ncols * A->K * sizeof(double);
  for (int sl = 0; sl < 4; ++sl)
    if ((rc = ensure_scratch(ctx, sl, sl < 2 ? vb : yb))) return rc;
  cudaStream_t st = ctx->stream;
  if (vb) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dbuf[0], v_re, vb, cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dbuf[1], v_im, vb, cudaMemcpyHostToDevice, st));
  }
  if (yb && T->nnz == 0) {
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->dbuf[2], 0, yb, st));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->dbuf[3], 0, yb, st));
  }
  SegScope scope{ctx};
  if ((rc = set_segments(ctx, A, order, threads))) return rc;
  if ((rc = launch_spmv(ctx, T, torder(order), ctx->dbuf[0], ctx->dbuf[1], ctx->dbuf[2], ctx->dbuf[3], st,
                        conjugate != 0)))
    return rc;
  if (yb) {
    CUDA_TRY(ctx, cudaMemcpyAsync(y_re, ctx->dbuf[2], yb, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(y_im, ctx->dbuf[3], yb, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return MPSG_OK;
}

int mpsg_cg(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t blen, const double* b,
            const double* x0, const mpsg_cg_config* cfg, double* x_out, double* history,
            int64_t history_cap, mpsg_cg_report* report) {
  if (!ctx || !A || !cfg || !report || !b) return MPSG_E_ARG;
  // SolverConfig::validate (krylov.hpp:69-75) and solver_init shape checks (:164-176)
  if (!(cfg->rel_tol > 0.0) || !(cfg->abs_tol > 0.0))
    return fail(ctx, MPSG_E_ARG, "solver: tolerances must be positive");
  if (cfg->max_iters < 1) return fail(ctx, MPSG_E_ARG, "solver: max_iters must be at least 1");
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "solver: complex matrices are not supported by cg");
  if (A->nrows != A->ncols)
    return fail(ctx, MPSG_E_DIM, "solver: operator must be square, got %lldx%lld", (long long)A->nrows,
                (long long)A->ncols);
  if (blen != A->ncols) return fail(ctx, MPSG_E_DIM, "solver: rhs length does not match the operator");
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "cg: unknown order %d", order);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  switch (A->K) {
    case 2: return run_cg<2>(ctx, A, order, b, x0, cfg, x_out, history, history_cap, report);
    case 3: return run_cg<3>(ctx, A, order, b, x0, cfg, x_out, history, history_cap, report);
    case 4: return run_cg<4>(ctx, A, order, b, x0, cfg, x_out, history, history_cap, report);
  }
  return fail(ctx, MPSG_E_ARG, "cg: unsupported K");
}

int mpsg_solve(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t blen, const double* b, const double* x0,
               const mpsg_solver_config* cfg, double* x_out, double* history, int64_t history_cap,
               mpsg_cg_report* report) {
  if (!ctx || !A || !cfg || !report || !b) return MPSG_E_ARG;
  // SolverConfig::validate (krylov.hpp:69-75) and solver_init shape checks (:164-176)
  if (!(cfg->rel_tol > 0.0) || !(cfg->abs_tol > 0.0))
    return fail(ctx, MPSG_E_ARG, "solver: tolerances must be positive");
  if (cfg->max_iters < 1) return fail(ctx, MPSG_E_ARG, "solver: max_iters must be at least 1");
  if (cfg->threads < 1) return fail(ctx, MPSG_E_ARG, "solver: threads must be at least 1");
  if (cfg->method < MPSG_CG || cfg->method > MPSG_GPBICG)
    return fail(ctx, MPSG_E_ARG, "solve: unknown method %d", cfg->method);
  if (cfg->dot_order != MPSG_DOT_TREE && cfg->dot_order != MPSG_DOT_SEQUENTIAL)
    return fail(ctx, MPSG_E_ARG, "solve: unknown dot order %d", cfg->dot_order);
  if (A->cplx) return fail(ctx, MPSG_E_ARG, "solver: complex matrices are not supported");
  if (A->nrows != A->ncols)
    return fail(ctx, MPSG_E_DIM, "solver: operator must be square, got %lldx%lld", (long long)A->nrows,
                (long long)A->ncols);
  if (blen != A->ncols) return fail(ctx, MPSG_E_DIM, "solver: rhs length does not match the operator");
  if (order < 0 || order > 2) return fail(ctx, MPSG_E_ARG, "solve: unknown order %d", order);
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  switch (A->K) {
    case 2: return krylov_driver<2>(ctx, A, nullptr, cfg, order, b, x0, x_out, history, history_cap, report);
    case 3: return krylov_driver<3>(ctx, A, nullptr, cfg, order, b, x0, x_out, history, history_cap, report);
    case 4: return krylov_driver<4>(ctx, A, nullptr, cfg, order, b, x0, x_out, history, history_cap, report);
  }
  return fail(ctx, MPSG_E_ARG, "solve: unsupported K");
}

int mpsg_partition_rows(const int64_t* indptr, int64_t nrows, int parts, int64_t* bounds) {
  // kernels.hpp:63-80: bounds[t] = first row with indptr >= total*t/parts
  if (!indptr || !bounds || parts < 1) return MPSG_E_ARG;
  for (int t = 0; t <= parts; ++t) bounds[t] = nrows;
  bounds[0] = 0;
  const int64_t total = indptr[nrows];
  for (int t = 1; t < parts; ++t) {
    const int64_t target = total * t / parts;
    int64_t lo = bounds[t - 1], hi = nrows;
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (indptr[mid] < target)
        lo = mid + 1;
      else
        hi = mid;
    }
    bounds[t] = lo;
  }
  return MPSG_OK;
}

uint64_t mpsg_checksum(int K, int64_t n, const double* v) {
  uint64_t h = 14695981039346656037ull;
  for (int64_t i = 0; i < n * K; ++i) {
    uint64_t bits;
    std::memcpy(&bits, v + i, 8);
    for (int b = 0; b < 8; ++b) {
      h ^= (bits >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

uint64_t mpsg_checksum_complex(int K, int64_t n, const double* re, const double* im) {
  return mpsg_checksum(K, n, re) * 1099511628211ull ^ mpsg_checksum(K, n, im);
}

}  // extern "C"
