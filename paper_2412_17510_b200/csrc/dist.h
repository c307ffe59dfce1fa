// dist.h -- row-sharded multi-GPU layer (one process per GPU, NCCL over
// NVLink/NVSwitch).  Internal to the library; the ABI is in include/mpsg.h.
//
// Shard rule: rank r owns the contiguous row block [bounds[r], bounds[r+1])
// chosen by the reference's partition_rows (kernels.hpp:63-80: equal nnz), and
// the matching block of x and y (square matrices).  Rows never split, so the
// exact orders (SCALAR / LANE4) stay bit-exact under any partition.
//
// Per SpMV the only traffic is the x halo: each rank needs the column interval
// [need_lo, need_hi) its rows touch; the parts owned by other ranks arrive by
// ncclSend/ncclRecv pairs in one group (neighbour halo for banded/stencil
// matrices, all-to-all blocks -- an allgather -- for unstructured ones) into a
// global-length x buffer indexed by global column, so the local kernels are
// the single-GPU kernels unchanged.
// Dot products in CG: each rank reduces its rows to one K-component partial,
// the partials are allgathered (P*K doubles) and summed in rank order with the
// multi-component add on every rank -- identical and deterministic everywhere
// (an ncclSum of doubles would destroy the multi-component exactness).
#pragma once
#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace mpsg {

// NCCL is resolved at run time (dlopen of libnccl.so.2, the library torch has
// usually loaded already), so single-GPU use never depends on it.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  static const NcclApi* get(std::string* err);
};

// Single-process group: one host thread per rank (each with its own
// mpsg_ctx, on one or several devices), data moved by device-to-device /
// peer copies ordered with CUDA events across the ranks' streams, and a host
// barrier to publish each collective's buffers and events.  No kernel ever
// waits on another rank's kernel (only stream-order dependencies), so ranks
// may share a GPU.  Used for single-process multi-GPU runs and to exercise the
// sharded path on one GPU.
struct LocalGroup {
  int P = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<const void*> ptr;       // per rank: buffer published for the collective
  std::vector<cudaEvent_t> ready;     // per rank: its buffer is complete
  std::vector<cudaEvent_t> consumed;  // per rank: its copies out of the others are done
  std::vector<int64_t> meta;          // per rank: 4 int64 (setup allgather)
  int refs = 0;
  void barrier();
};

}  // namespace mpsg

struct mpsg_comm {
  mpsg_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  const mpsg::NcclApi* api = nullptr;
  mpsg::LocalGroup* local = nullptr;  // single-process group backend (instead of NCCL)
};

struct mpsg_dcsr {
  mpsg_comm* comm = nullptr;
  mpsg_csr* local = nullptr;  // this rank's rows, global column indices
  // the same rows split for the halo overlap: interior rows (every column in
  // this rank's block) run while the halo moves, boundary rows after it
  mpsg_csr* local_int = nullptr;
  mpsg_csr* local_bnd = nullptr;
  int64_t n_interior = 0;
  int K = 2;
  bool cplx = false;
  int64_t nglobal = 0, row_begin = 0, row_end = 0;
  std::vector<int64_t> bounds;  // [nranks+1] row ownership
  std::vector<int64_t> need;    // [2*nranks] column interval each rank reads
  std::vector<int64_t> send;    // [2*nranks] my rows peer q reads (lo, hi)
  std::vector<int64_t> recv;    // [2*nranks] q's rows I read (lo, hi)
  double* xfull[2] = {nullptr, nullptr};  // global-length x (re, im)
  double* ybuf[2] = {nullptr, nullptr};   // local y scratch (host-pointer calls)
  int64_t halo_rows = 0;                  // rows received per SpMV
};

namespace mpsg {

#define NCCL_TRY(cm, call)                                                                  \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail((cm)->ctx, MPSG_E_NCCL, "%s: %s", #call, (cm)->api->GetErrorString(r_)); \
  } while (0)

// Exchange the halo of a global-length buffer whose own block is in place.
int halo_exchange(const mpsg_dcsr* A, double* xfull, cudaStream_t st);
// y = A x for a sharded matrix, x's own block in place in the global-length
// xfull buffers: interior rows on ctx->side concurrently with the halo
// exchange, then boundary rows (or halo + all rows when not split).
int dist_spmv(const mpsg_dcsr* A, int order, double* xre, double* xim, double* yre, double* yim, cudaStream_t st);
// out[P*K] = every rank's in[K] (rank order).
int allgather_mc(const mpsg_comm* c, const double* in, double* out, int K, cudaStream_t st);
// Host allgather of n int64 per rank (setup only).
int allgather_host(const mpsg_comm* c, const int64_t* mine, int64_t* all, int n);

// Distributed device CG (cg_inst.cuh), b / x0 / x_out are this rank's block.
template <int K>
int run_dcg(mpsg_dcsr* A, int order, const double* b_host, const double* x0, const mpsg_cg_config* cfg,
            double* x_out, double* history, int64_t history_cap, mpsg_cg_report* rep);

}  // namespace mpsg
