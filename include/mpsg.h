/*
 * mpsg.h -- C ABI of the B200-native multi-precision sparse path.
 *
 * Drop-in boundary for the reference's hot path (paths under
 * /root/reference/proj/include/mps/):
 *
 *   reference entry point (file:line)                       replaced by
 *   ------------------------------------------------------  ----------------------
 *   CsrMatrix<E> / CsrValues<MultiComponent<K>>             mpsg_csr_upload
 *       (sparse.hpp:47-78; convert_csr sparse.hpp:195-207)
 *   ComplexSparseMatrix<E> (sparse.hpp:221-230)             mpsg_csr_upload(is_complex=1)
 *   spmv<E,F>(A, v, KernelMode) (kernels.hpp:348-366)       mpsg_spmv / mpsg_spmv_dev
 *   spmv_complex<E,F>(A, v, KernelMode) (kernels.hpp:399)   mpsg_spmv_complex(_dev)
 *   CsrOperator<E>::apply (krylov.hpp:101-120)              mpsg_spmv_dev (operator seam)
 *   solve_cg<E,Op>(op, b, SolverConfig) (krylov.hpp:238)    mpsg_cg
 *   solve<E,Op>(op, b, SolverConfig) (krylov.hpp:596-606)   mpsg_solve
 *     (solve_bicg / _cgs / _bicgstab / _gpbicg, :283-594)
 *   detail::partition_rows (kernels.hpp:63-80)              mpsg_partition_rows
 *   checksum (bench.hpp:113-150)                            mpsg_checksum(_complex)
 *
 * Conventions.
 *  - K is the component count: 2 (double-double), 3 (triple-double),
 *    4 (quad-double).
 *  - Vectors are AoS: element i occupies doubles [i*K, i*K+K), which is the
 *    memory image of std::vector<MultiComponent<K>> (MultiComponent<K> is a
 *    std::array<double,K>, multicomp.hpp:17-30), so `v.data()` can be passed
 *    as `const double*`.
 *  - Matrix values are K component planes, planes[j][k] = component j of
 *    nonzero k (CsrValues::component(j), sparse.hpp:63); complex matrices pass
 *    2K planes (re components then im components) over one shared structure.
 *  - Indices are int64 as in the reference (sparse.hpp:73-74); the device
 *    keeps int32 and rejects anything that does not fit (MPSG_E_RANGE).
 *  - order: MPSG_ORDER_SCALAR reproduces `lanes_enabled = false`
 *    (row_sum_scalar, kernels.hpp:90-99) bit for bit; MPSG_ORDER_LANE4
 *    reproduces the reference default `lanes_enabled = true`
 *    (row_sum_lanes_pure, kernels.hpp:103-121) bit for bit; MPSG_ORDER_FAST
 *    reorders long-row accumulation and fuses each product-accumulate (one
 *    renormalisation per nonzero, TD/QD/DD) for throughput, and is checked
 *    against the componentwise bound |y - y_ref| <= 4 * rowlen * u * sum|a||x|.
 *    KernelMode::threads has no device meaning and is ignored.
 *  - Errors are returned as status codes; nothing crosses the ABI as an
 *    exception.  mpsg_last_error(ctx) gives the message (for MPSG_E_DIM it is
 *    the reference's std::invalid_argument text, kernels.hpp:333-339).
 *  - A context is bound to one device and is not thread-safe (one host thread
 *    per context).  Host-pointer calls are synchronous like the reference;
 *    *_dev calls are stream-ordered and asynchronous.
 */
#ifndef MPSG_H
#define MPSG_H

#include <stdint.h>

#if defined(_WIN32)
#define MPSG_API
#else
#define MPSG_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MPSG_VERSION_MAJOR 0
#define MPSG_VERSION_MINOR 1

enum mpsg_status {
  MPSG_OK = 0,
  MPSG_E_DIM = 1,    /* vector / matrix dimension mismatch (std::invalid_argument) */
  MPSG_E_RANGE = 2,  /* index does not fit int32, or out of [0, ncols) */
  MPSG_E_CUDA = 3,   /* CUDA runtime failure */
  MPSG_E_NCCL = 4,   /* reserved for the multi-GPU layer */
  MPSG_E_OOM = 5,    /* device allocation failed */
  MPSG_E_ARG = 6,    /* invalid argument (K, order, null pointer, config) */
  MPSG_E_STRUCT = 7  /* malformed CSR (indptr not monotone / wrong length) */
};

enum mpsg_order {
  MPSG_ORDER_SCALAR = 0, /* lanes off: bit-exact with the reference */
  MPSG_ORDER_LANE4 = 1,  /* lanes on (reference default): bit-exact */
  MPSG_ORDER_FAST = 2    /* throughput: long rows reordered, fused product-accumulates (bounded error) */
};

/* SolverStatus, krylov.hpp:46 */
enum mpsg_solver_status {
  MPSG_CONVERGED = 0,
  MPSG_MAX_ITERATIONS = 1,
  MPSG_BREAKDOWN = 2,
  MPSG_DIVERGED = 3
};

/* KrylovMethod, krylov.hpp:24 (same order) */
enum mpsg_method {
  MPSG_CG = 0,
  MPSG_BICG = 1,
  MPSG_CGS = 2,
  MPSG_BICGSTAB = 3,
  MPSG_GPBICG = 4
};

/* Dot-product order of the device solvers. */
enum mpsg_dot_order {
  MPSG_DOT_TREE = 0,       /* fixed-shape parallel tree: deterministic, not the reference's bits */
  MPSG_DOT_SEQUENTIAL = 1  /* one thread, i ascending: the reference's dot (krylov.hpp:122-128);
                              with an exact SpMV order the solve reproduces the reference bit for bit */
};

/* mpsg_csr_upload_ex flags */
enum mpsg_csr_flags {
  MPSG_CSR_COMPLEX = 1,   /* 2x the planes: re then im over one structure (ComplexSparseMatrix) */
  MPSG_CSR_MIXED = 2,     /* binary64 values: 1 plane (2 complex), vectors in K components
                             (CsrMatrix<double> x MultiComponent<K>, the paper's "M" mode) */
  MPSG_CSR_TRANSPOSE = 4  /* also build the device transpose for mpsg_sptmv* */
};

typedef struct mpsg_ctx mpsg_ctx;
typedef struct mpsg_csr mpsg_csr;

/* Layout statistics of an uploaded matrix. */
typedef struct mpsg_csr_stats {
  int64_t nrows, ncols, nnz;
  int32_t K, is_complex;
  int64_t nslices;         /* SELL slices (short rows) */
  int64_t sell_elems;      /* padded SELL elements */
  int64_t nlong;           /* rows in the long-row store */
  int64_t long_nnz;        /* nonzeros in the long-row store */
  int64_t nchunks;         /* fast-mode warp chunks over long rows */
  int64_t device_bytes;    /* device memory held by the matrix (and its transpose) */
  int32_t is_mixed;        /* binary64 values */
  int32_t has_transpose;   /* uploaded with MPSG_CSR_TRANSPOSE */
} mpsg_csr_stats;

/* SolverConfig subset used by CG (krylov.hpp:58-75). */
typedef struct mpsg_cg_config {
  double rel_tol;     /* default 1e-13 */
  double abs_tol;     /* default 1e-99 */
  int64_t max_iters;  /* default 10000 */
  int32_t check_every; /* host polls the device status every N iterations (0 = 32) */
  int32_t use_graph;   /* capture the iteration batch in a CUDA graph (default 1) */
  int32_t variant;     /* mpsg_cg_variant (0 = auto) */
  int32_t reserved;
} mpsg_cg_config;

/* CG iteration form.  CLASSIC is the reference's (krylov.hpp:238-281: two dot
 * products per iteration); ONE_REDUCTION is the Chronopoulos-Gear recurrence
 * with the same Krylov iterates and a single fused reduction (<r,r>, <Ar,r>)
 * per iteration -- one allgather per iteration when the rows are sharded.
 * AUTO: CLASSIC on one GPU, ONE_REDUCTION for mpsg_dcg over more than one rank. */
typedef enum mpsg_cg_variant { MPSG_CG_AUTO = 0, MPSG_CG_CLASSIC = 1, MPSG_CG_ONE_REDUCTION = 2 } mpsg_cg_variant;

/* SolverConfig (krylov.hpp:58-75) for mpsg_solve. */
typedef struct mpsg_solver_config {
  int32_t method;      /* mpsg_method (the reference default is BiCGSTAB) */
  int32_t threads;     /* KernelMode::threads of the operator: BiCG's sptmv merge order */
  double rel_tol;      /* default 1e-13 */
  double abs_tol;      /* default 1e-99 */
  int64_t max_iters;   /* default 10000 */
  int32_t check_every; /* host polls the device status every N iterations (0 = 32) */
  int32_t use_graph;   /* capture the iteration batch in a CUDA graph (default 1) */
  int32_t dot_order;   /* mpsg_dot_order */
  int32_t reserved;
} mpsg_solver_config;

/* SolverReport (krylov.hpp:77-88). */
typedef struct mpsg_cg_report {
  int32_t status; /* mpsg_solver_status */
  int32_t converged;
  int64_t iterations;
  int64_t history_len; /* entries written to the caller's history buffer */
  double rhs_norm;
  double final_recurrence_residual;
  double final_true_residual;
  double setup_seconds;
  double solve_seconds;   /* host wall clock of the iteration loop (as the reference) */
  char detail[64];
  double device_seconds;  /* the same loop timed with CUDA events on the solve stream */
} mpsg_cg_report;

/* ---- context --------------------------------------------------------- */
MPSG_API int mpsg_ctx_create(int device, mpsg_ctx** out);
/* Why the last mpsg_ctx_create on this host thread failed ("" if it did not):
 * the CUDA error name and text.  A device held by another process
 * (cudaErrorDevicesUnavailable) is retried inside mpsg_ctx_create for ~2 s. */
MPSG_API const char* mpsg_create_error(void);
MPSG_API void mpsg_ctx_destroy(mpsg_ctx* ctx);
MPSG_API const char* mpsg_last_error(const mpsg_ctx* ctx);
/* Use a caller-owned cudaStream_t (as void*) for subsequent work; NULL
 * restores the context's own stream. */
MPSG_API int mpsg_ctx_set_stream(mpsg_ctx* ctx, void* stream);
/* Tunables (0 keeps the default): long-row threshold (256), SELL sort window
 * (16384 rows), fast-mode chunk length (2048). Affect later uploads. */
MPSG_API int mpsg_ctx_set_layout(mpsg_ctx* ctx, int64_t long_threshold, int64_t sigma, int64_t fast_chunk);
/* Block until all work queued on the context's stream has finished. */
MPSG_API int mpsg_ctx_synchronize(mpsg_ctx* ctx);

/* ---- matrices -------------------------------------------------------- */
/* Copies a host CSR (reference layout) to the device once.  planes has K
 * (real) or 2K (complex) entries, each nnz = indptr[nrows] doubles. */
MPSG_API int mpsg_csr_upload(mpsg_ctx* ctx, int K, int is_complex, int64_t nrows, int64_t ncols,
                    const int64_t* indptr, const int64_t* indices, const double* const* planes,
                    mpsg_csr** out);
/* General form: flags from mpsg_csr_flags; planes has K (Pure) or 1 (Mixed)
 * entries per part, times 2 for complex. */
MPSG_API int mpsg_csr_upload_ex(mpsg_ctx* ctx, int K, int flags, int64_t nrows, int64_t ncols,
                                const int64_t* indptr, const int64_t* indices, const double* const* planes,
                                mpsg_csr** out);
MPSG_API void mpsg_csr_destroy(mpsg_csr* A);
MPSG_API int mpsg_csr_get_stats(const mpsg_csr* A, mpsg_csr_stats* out);

/* ---- SpMV (kernels.hpp:348-366, 399-416) ------------------------------ */
/* Host pointers, synchronous: y[nrows*K] = A x[xlen*K]. */
MPSG_API int mpsg_spmv(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t xlen, const double* x,
              double* y);
/* Device pointers, asynchronous on `stream` (NULL: the context stream).
 * DD / QD device vectors must be 16-byte aligned (every cudaMalloc pointer and
 * every element offset into one is; TD: 8 bytes) -- MPSG_E_ARG otherwise.  A
 * 32-byte aligned QD x is gathered with 256-bit loads. */
MPSG_API int mpsg_spmv_dev(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* d_x, double* d_y,
                  void* stream);
MPSG_API int mpsg_spmv_complex(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t xlen,
                      const double* x_re, const double* x_im, double* y_re, double* y_im);
MPSG_API int mpsg_spmv_complex_dev(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* d_x_re,
                          const double* d_x_im, double* d_y_re, double* d_y_im, void* stream);

/* ---- transposed products (kernels.hpp:368-394, 419-441) ---------------- */
/* y[ncols*K] = A^T v[nrows*K]; needs MPSG_CSR_TRANSPOSE at upload.  The
 * exact orders reproduce the reference sptmv at one thread (bit for bit, lanes
 * on or off -- the lane batches there are per-element exact); FAST reorders
 * long columns. */
MPSG_API int mpsg_sptmv(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t vlen, const double* v, double* y);
MPSG_API int mpsg_sptmv_dev(mpsg_ctx* ctx, const mpsg_csr* A, int order, const double* d_v, double* d_y,
                            void* stream);
/* The reference sptmv at `threads` OpenMP threads: per-thread accumulators
 * over partition_rows(threads) row blocks merged in thread order
 * (kernels.hpp:368-394) -- thread-count dependent bits, reproduced exactly in
 * the exact orders (threads <= 1: as mpsg_sptmv). */
MPSG_API int mpsg_sptmv_ex(mpsg_ctx* ctx, const mpsg_csr* A, int order, int threads, int64_t vlen,
                           const double* v, double* y);
/* conjugate != 0: the adjoint A^H v (y.re = rr + ii, y.im = ri - ir). */
MPSG_API int mpsg_sptmv_complex(mpsg_ctx* ctx, const mpsg_csr* A, int order, int conjugate, int64_t vlen,
                                const double* v_re, const double* v_im, double* y_re, double* y_im);
MPSG_API int mpsg_sptmv_complex_ex(mpsg_ctx* ctx, const mpsg_csr* A, int order, int threads, int conjugate,
                                   int64_t vlen, const double* v_re, const double* v_im, double* y_re,
                                   double* y_im);
MPSG_API int mpsg_sptmv_complex_dev(mpsg_ctx* ctx, const mpsg_csr* A, int order, int conjugate,
                                    const double* d_v_re, const double* d_v_im, double* d_y_re, double* d_y_im,
                                    void* stream);

/* ---- conjugate gradient (krylov.hpp:238-281) -------------------------- */
/* Device-resident CG on A (real, square).  b and x0 (NULL = zero start) are
 * host AoS vectors of length nrows; x_out receives the iterate; history
 * receives ||r_k|| for k = 0.. (up to history_cap entries). */
MPSG_API int mpsg_cg(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t blen, const double* b,
            const double* x0, const mpsg_cg_config* cfg, double* x_out, double* history,
            int64_t history_cap, mpsg_cg_report* report);

/* ---- solve() (krylov.hpp:596-606): CG, BiCG, CGS, BiCGSTAB, GPBiCG --- */
/* Device-resident Krylov solve of A x = b (real, square), the method chosen
 * by cfg->method; the reference solver's breakdown / divergence / half-step
 * exits, iteration counts, residual history and final true residual.  BiCG
 * needs the transpose (MPSG_CSR_TRANSPOSE).  Arguments as mpsg_cg; the
 * report's detail is the reference text ("bicgstab: omega vanished", ...). */
MPSG_API int mpsg_solve(mpsg_ctx* ctx, const mpsg_csr* A, int order, int64_t blen, const double* b,
                        const double* x0, const mpsg_solver_config* cfg, double* x_out, double* history,
                        int64_t history_cap, mpsg_cg_report* report);

/* ---- row-sharded multi-GPU (one process per GPU, NCCL) ------------------ */
/* Rank r owns rows [bounds[r], bounds[r+1]) (mpsg_partition_rows gives the
 * reference's equal-nnz rule, kernels.hpp:63-80) and the same block of x and
 * y; per SpMV only the x halo moves (ncclSend/ncclRecv, NVLink/NVSwitch); CG
 * dot products are allgathered per-rank partials summed in rank order.  The
 * exact orders stay bit-exact for any partition. */
typedef struct mpsg_comm mpsg_comm;
typedef struct mpsg_dcsr mpsg_dcsr;
/* NCCL unique id (128 bytes) created on one rank and broadcast by the caller. */
MPSG_API int mpsg_comm_unique_id(unsigned char* id);
/* id may be NULL when nranks == 1.  NCCL is loaded at run time (libnccl.so.2). */
MPSG_API int mpsg_comm_create(mpsg_ctx* ctx, int nranks, int rank, const unsigned char* id, mpsg_comm** out);
/* Single-process group of nranks ranks, one mpsg_ctx each (same or different
 * devices): collectives are device/peer copies ordered by CUDA events across
 * the ranks' streams, no NCCL.  Every rank must be driven by its own host
 * thread (the collectives rendezvous through a host barrier).  out[r] gets
 * rank r's handle. */
MPSG_API int mpsg_comm_create_local(mpsg_ctx* const* ctxs, int nranks, mpsg_comm** out);
MPSG_API void mpsg_comm_destroy(mpsg_comm* comm);
/* This rank's rows [row_begin, row_end) of a square nglobal x nglobal matrix:
 * indptr rebased (row_end-row_begin+1 entries), global column indices, K or
 * 2K planes.  Collective: builds the halo plan with every rank. */
MPSG_API int mpsg_dcsr_upload(mpsg_comm* comm, int K, int is_complex, int64_t nglobal, int64_t row_begin,
                              int64_t row_end, const int64_t* indptr, const int64_t* indices,
                              const double* const* planes, mpsg_dcsr** out);
MPSG_API void mpsg_dcsr_destroy(mpsg_dcsr* A);
/* bounds: nranks+1 entries (may be NULL); halo_rows: rows received per SpMV. */
MPSG_API int mpsg_dcsr_info(const mpsg_dcsr* A, int64_t* bounds, int64_t* halo_rows);
/* Rows of this rank whose columns all lie in its own block: they run while
 * the x halo moves (0 when the rows are not split, e.g. one rank). */
MPSG_API int mpsg_dcsr_interior_rows(const mpsg_dcsr* A, int64_t* interior_rows);
/* y_local = (A x)[row block]; x_local / y_local are this rank's blocks.
 * Collective (every rank calls it with the same order). */
MPSG_API int mpsg_dspmv(mpsg_dcsr* A, int order, const double* x_local, double* y_local);
MPSG_API int mpsg_dspmv_dev(mpsg_dcsr* A, int order, const double* d_x_local, double* d_y_local, void* stream);
MPSG_API int mpsg_dspmv_complex_dev(mpsg_dcsr* A, int order, const double* d_xr_local, const double* d_xi_local,
                                   double* d_yr_local, double* d_yi_local, void* stream);
/* Row-sharded CG (krylov.hpp:238-281); b / x0 / x_out are this rank's blocks,
 * the history and report are identical on every rank.  Collective. */
MPSG_API int mpsg_dcg(mpsg_dcsr* A, int order, const double* b_local, const double* x0_local,
                      const mpsg_cg_config* cfg, double* x_out_local, double* history, int64_t history_cap,
                      mpsg_cg_report* report);
/* Row-sharded solve() (krylov.hpp:596-606) for CG, CGS, BiCGSTAB and GPBiCG
 * (BiCG's transposed product is not sharded: MPSG_E_ARG); arguments as
 * mpsg_dcg, method / dot order in cfg.  Dots are per-rank partials summed in
 * rank order, so the sequential dot order is the reference's only at P = 1.
 * Collective. */
MPSG_API int mpsg_dsolve(mpsg_dcsr* A, int order, const double* b_local, const double* x0_local,
                         const mpsg_solver_config* cfg, double* x_out_local, double* history, int64_t history_cap,
                         mpsg_cg_report* report);
/* Host-only halo plan: for every peer q, the interval of my rows q reads
 * (send[2q], send[2q+1]) and of q's rows I read (recv[...]); need[2q..] is
 * the column interval rank q reads.  Empty intervals are (0, 0). */
MPSG_API int mpsg_halo_plan(int nranks, int rank, const int64_t* bounds, const int64_t* need, int64_t* send,
                            int64_t* recv);

/* ---- host utilities ---------------------------------------------------- */
/* nnz-balanced contiguous row bounds (kernels.hpp:63-80), parts+1 entries. */
MPSG_API int mpsg_partition_rows(const int64_t* indptr, int64_t nrows, int parts, int64_t* bounds);
/* FNV-1a over component bits in AoS order (bench.hpp:113-150). */
MPSG_API uint64_t mpsg_checksum(int K, int64_t n, const double* v);
MPSG_API uint64_t mpsg_checksum_complex(int K, int64_t n, const double* re, const double* im);
MPSG_API const char* mpsg_version(void);

/* The reference harness's input vectors (make_vector / make_complex_vector,
 * bench.hpp:78-111), computed with the device ops (the reference's bits):
 * im == NULL: re[j] = sqrt(2) * (j+1); else re + i im = sqrt(2 + 3i) * (j+1). */
MPSG_API int mpsg_make_vector(mpsg_ctx* ctx, int K, int64_t n, double* re, double* im);

/* ---- measurement / verification -------------------------------------- */
/* fp64-pipe throughput (DFMA instructions per second) on the context device:
 * the roofline denominator for the fp64-bound TD/QD configurations. */
MPSG_API int mpsg_measure_fp64_peak(mpsg_ctx* ctx, double* ops_per_s);
/* Batched device multi-component op on AoS device arrays (n elements of K):
 * op 0 add, 1 mul, 2 mul_by_double(a, b[i][0]), 3 sub, 4 divide, 5 sqrt(a)
 * (multicomp.hpp:225-322).  Asynchronous on the context stream. */
MPSG_API int mpsg_mc_op_dev(mpsg_ctx* ctx, int op, int K, int64_t n, const double* d_a,
                            const double* d_b, double* d_out);

#ifdef __cplusplus
}
#endif

#endif /* MPSG_H */
