// internal.h -- host-side internals shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/mpsg.h"
#include "layout.h"

using mpsg::LongView;
using mpsg::SellView;

struct mpsg_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // current (own or caller's)
  cudaStream_t aux = nullptr;     // long-row kernels run here, forked/joined by events
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t copy = nullptr;    // device->host copies overlapped with SpMV parts
  cudaStream_t side = nullptr;    // sharded SpMV: interior rows while the x halo moves
  cudaEvent_t ev_side0 = nullptr, ev_side1 = nullptr;
  cudaEvent_t ev_part[16] = {};
  bool overlap = true;            // MPSG_OVERLAP=0 disables
  // transposed product at T > 1 threads: segment bounds of the running call
  // (set by mpsg_sptmv*_ex around the launch; seg_T == 1 means off)
  int64_t* seg_bounds = nullptr;
  size_t seg_cap = 0;
  int seg_T = 1;
  std::vector<int64_t> seg_host;
  std::string err;
  // pinned staging for pageable host vectors (two chunk slots, double-buffered
  // against the DMA; the host side copies with OpenMP threads)
  double* hslot[2] = {nullptr, nullptr};
  size_t hslot_cap = 0;
  cudaEvent_t hslot_ev[2] = {nullptr, nullptr};
  bool stage_host = true;         // MPSG_STAGE_HOST=0 disables
  // scratch for host-pointer calls
  double* dbuf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t dcap[4] = {0, 0, 0, 0};
  // L2 residency for the gathered vector: launches carry an access-policy
  // window over x (persisting) so the streamed matrix (evict-first loads)
  // does not push x out of L2.  persist_max = the device's persisting-L2
  // capacity (0: unsupported / disabled by MPSG_L2_PERSIST=0).
  size_t persist_max = 0;
  int64_t long_threshold = 256;
  int64_t sigma = 16384;
  int64_t fast_chunk = 2048;
  // column blocking of long-row chunks (fast order): rows of at least
  // colblock_min elements are cut where their columns cross a multiple of
  // colblock_bytes worth of x; 0 disables.
  int64_t colblock_bytes = 16ll << 20;
  int64_t colblock_min = 4096;
};

struct mpsg_csr {
  int K = 2;
  bool cplx = false;
  bool mixed = false;         // binary64 values (Mixed mode, kernels.hpp:55-58)
  mpsg_csr* trans = nullptr;  // device transpose, for the transposed products
  std::vector<int64_t> host_indptr;  // A's row pointer (kept with the transpose: thread partition)
  int64_t nrows = 0, ncols = 0, nnz = 0;
  // SELL store
  int C = 32;
  int64_t nslices = 0, sell_elems = 0;
  int64_t* slice_ptr = nullptr;
  int* slot_row = nullptr;
  int* slot_len = nullptr;
  int* scol = nullptr;
  double* sval = nullptr;
  // long store
  int64_t nlong = 0, long_nnz = 0, nchunks = 0, chunk = 2048;
  int* lrow = nullptr;
  int64_t* lptr = nullptr;
  int* lcol = nullptr;
  double* lval = nullptr;
  int* chunk_row = nullptr;
  int64_t* chunk_beg = nullptr;
  int64_t* chunk_end = nullptr;
  int* chunk_slot = nullptr;
  int* chunk_first = nullptr;
  double* partial = nullptr;
  unsigned* counter = nullptr;
  // real TD only: x re-laid out to 32 bytes per element ([ncols][4], last
  // double unused) before the FAST short-row kernel, so that every gather is
  // one aligned 256-bit load = one L1 wavefront instead of three 64-bit ones
  double* xpad = nullptr;
  int64_t device_bytes = 0;
  // host-call output parts: slices [part_slice[p], part_slice[p+1]) write rows
  // [part_row[p], part_row[p+1]) (besides long rows); empty = no overlap
  std::vector<int64_t> part_slice, part_row;

  SellView sell() const {
    return SellView{(int)nslices, C, slice_ptr, slot_row, slot_len, scol, sval, sell_elems};
  }
  // the slices [s0, s1) as a view (slice_ptr values are absolute offsets)
  SellView sell_range(int64_t s0, int64_t s1) const {
    return SellView{(int)(s1 - s0), C, slice_ptr + s0, slot_row + s0 * C, slot_len + s0 * C, scol, sval,
                    sell_elems};
  }
  LongView lng() const {
    return LongView{(int)nlong, lrow, lptr, lcol, lval, long_nnz, (int)chunk, (int)nchunks,
                    chunk_row, chunk_beg, chunk_end, chunk_slot, chunk_first, partial, counter};
  }
};

namespace mpsg {

inline int fail(mpsg_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

#define CUDA_TRY(ctx, call)                                                                   \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? MPSG_E_OOM : MPSG_E_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
  } while (0)

// Launch `kern` with an L2 access-policy window over [win, win+win_bytes)
// when the context enables it (the window travels with the launch, so it is
// captured into CUDA graphs too).
template <class... KArgs, class... Args>
cudaError_t launch_win(const mpsg_ctx* ctx, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, const void* win, size_t win_bytes, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (ctx->persist_max > 0 && win && win_bytes > 0) {
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(win);
    attr[0].val.accessPolicyWindow.num_bytes = win_bytes;
    attr[0].val.accessPolicyWindow.hitRatio =
        win_bytes <= ctx->persist_max ? 1.0f : (float)ctx->persist_max / (float)win_bytes;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// SpMV launch for one (K, complex) instantiation (spmv_k{2,3,4}.cu).
template <int K, bool CPLX>
int launch_spmv_k(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* xre,
                  const double* xim, double* yre, double* yim, cudaStream_t st, bool conj, int part = -2);
// Dispatch over K / complex (capi.cu).  conj: complex combine of the adjoint
// (y.re = rr + ii, y.im = ri - ir).
int launch_spmv(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* xre, const double* xim,
                double* yre, double* yim, cudaStream_t st, bool conj = false);
// Pieces of one SpMV: part < 0 launches the long-row kernel only (on `st`);
// part >= 0 the SELL slices of output part `part` (A->part_slice).
int launch_spmv_part(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* xre, const double* xim,
                     double* yre, double* yim, cudaStream_t st, bool conj, int part);
// Output rows of an uploaded matrix renumbered: row i of the uploaded CSR
// writes y[map[i]] (a row subset of a larger matrix; capi.cu).
int remap_rows(mpsg_ctx* ctx, mpsg_csr* A, const std::vector<int>& map);
// Device CG driver for one K (cg_k{2,3,4}.cu).
template <int K>
int run_cg(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* b_host, const double* x0,
           const mpsg_cg_config* cfg, double* x_out, double* history, int64_t history_cap,
           mpsg_cg_report* rep);

// Device solve() driver for one K (krylov_k{2,3,4}.cu).
template <int K>
int krylov_driver(mpsg_ctx* ctx, const mpsg_csr* A, const mpsg_dcsr* D, const mpsg_solver_config* cfg, int order,
                  const double* b_host, const double* x0_host, double* x_out, double* history,
                  int64_t history_cap, mpsg_cg_report* rep);
// Segment bounds of the reference's T-thread sptmv (partition_rows of A's
// rows, kernels.hpp:368-394) for the transposed launches that follow
// (ctx->seg_T; threads <= 1 or FAST turns it off).
int set_segments(mpsg_ctx* ctx, const mpsg_csr* A, int order, int threads);

}  // namespace mpsg
