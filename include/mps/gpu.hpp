// mps/gpu.hpp -- C++ drop-in for the reference's SpMV / SpTMV / CG path on B200.
//
// Header-only layer over the C ABI in mpsg.h (libmpsg.so).  It takes and
// returns the reference's own types, so a caller of the reference
// (/root/reference/proj/include/mps/) switches by changing the namespace:
//
//   reference (file:line)                                  drop-in here
//   -----------------------------------------------------  -----------------------------------
//   mps::spmv(const CsrMatrix<E>&, const std::vector<F>&,  mps::gpu::spmv (same signature)
//             const KernelMode&)        kernels.hpp:348
//   mps::sptmv(...)                     kernels.hpp:368    mps::gpu::sptmv (same signature)
//   mps::spmv_complex(const ComplexSparseMatrix<E>&,       mps::gpu::spmv_complex (same)
//             const ComplexVector<F>&, const KernelMode&)  kernels.hpp:399
//   mps::sptmv_complex(..., bool conjugate) kernels.hpp:419 mps::gpu::sptmv_complex (same)
//   mps::CsrOperator<E> (Op concept)    krylov.hpp:101     mps::gpu::GpuCsrOperator<E>
//   mps::solve_cg(op, b, cfg)           krylov.hpp:238     mps::gpu::solve_cg (device-resident)
//   mps::solve(op, b, cfg) and          krylov.hpp:596     mps::gpu::solve / solve_bicg / solve_cgs /
//     solve_bicg/cgs/bicgstab/gpbicg    krylov.hpp:283-594   solve_bicgstab / solve_gpbicg (device-
//                                                            resident; DotOrder::Sequential = the
//                                                            reference's bits)
//                                                          -- or the reference's own solvers
//                                                          (solve_cg, solve_bicg, ...) with a
//                                                          GpuCsrOperator (same Op concept)
//   mps::detail::partition_rows         kernels.hpp:63     mps::gpu::partition_rows
//   mps::checksum                       bench.hpp:113      (unchanged; results are host vectors)
//
// Element types (kernels.hpp:50-60): Pure mode, E = F = MultiComponent<K>
// (K = 2, 3, 4); Mixed mode, E = double and F = MultiComponent<K> (the
// paper's "M": binary64 matrix, product mul_by_double(v, a)).  Other types
// (binary64 x binary64, BigFloat) fail to compile: there is no CPU fallback.
//
// Include the reference headers first (this file uses mps::CsrMatrix,
// MultiComponent, KernelMode, SolverConfig, SolveResult, ...), then this one;
// link libmpsg.so.  Semantics kept from the reference:
//  * KernelMode::lanes_enabled selects the accumulation order, reproduced bit
//    for bit (true: row_sum_lanes_*, kernels.hpp:103-142; false:
//    row_sum_scalar, kernels.hpp:90).  KernelMode::threads has no device
//    meaning for spmv and is ignored; sptmv reproduces the reference at that
//    thread count (its per-thread accumulators are merged in thread order;
//    lanes do not change its bits).  The overloads taking
//    mps::gpu::Order::Fast select the throughput order (componentwise error
//    bound instead of bits).
//  * dimension errors throw std::invalid_argument with the reference message
//    (kernels.hpp:333-339); solver breakdown / divergence are reported in
//    SolverReport, never thrown (krylov.hpp:46, 203-213).
//  * host-vector calls are synchronous, like the reference.
//
// The reference-signature drop-ins upload a matrix once and cache it, keyed
// by its address, buffer pointers, shape and a content fingerprint (a hash of
// up to 2 x 1024 evenly spaced entries of indptr, indices and every value
// plane, plus the first and last of each).  A matrix destroyed and rebuilt at
// the same address with the same buffers is therefore caught unless the two
// agree on every sampled entry; at most kCacheEntries matrices per element
// type stay resident (least recently used evicted).  A caller that rewrites
// values in place between calls -- which the sample can miss -- must call
// mps::gpu::invalidate(A), or hold an explicit DeviceCsr (no cache at all).
#pragma once

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

#include "../mpsg.h"

namespace mps {
namespace gpu {

namespace detail {
template <class T>
struct mc_width : std::integral_constant<int, 0> {};
template <int K>
struct mc_width<MultiComponent<K>> : std::integral_constant<int, K> {};

// (matrix element, vector element) pairs the device runs
template <class E, class F>
struct device_pair : std::false_type {};
template <int K>
struct device_pair<MultiComponent<K>, MultiComponent<K>> : std::true_type {};  // Pure
template <int K>
struct device_pair<double, MultiComponent<K>> : std::true_type {};  // Mixed

inline void raise(mpsg_ctx* ctx, int rc) {
  if (rc == MPSG_OK) return;
  std::string msg = mpsg_last_error(ctx);
  if (rc == MPSG_E_DIM) throw std::invalid_argument(msg);
  throw std::runtime_error("mpsg error " + std::to_string(rc) + ": " + msg);
}

inline std::string dim_msg(const char* what, std::size_t v, std::int64_t m) {  // kernels.hpp:333-339
  return std::string(what) + ": vector length " + std::to_string(v) + " does not match matrix dimension " +
         std::to_string(m);
}

// value planes of one CsrMatrix part: K SoA planes (Pure), or the binary64 array (Mixed)
template <int K>
void planes_of(const CsrMatrix<MultiComponent<K>>& A, const double** out) {
  for (int j = 0; j < K; ++j) out[j] = A.values.component(j);  // sparse.hpp:63
}
inline void planes_of(const CsrMatrix<double>& A, const double** out) { out[0] = A.values.data(); }
template <int K>
constexpr int nplanes(const CsrMatrix<MultiComponent<K>>*) { return K; }
constexpr int nplanes(const CsrMatrix<double>*) { return 1; }
}  // namespace detail

// ---------------------------------------------------------------- context
class Context {
 public:
  explicit Context(int device = 0) {
    int rc = mpsg_ctx_create(device, &ctx_);
    if (rc != MPSG_OK) throw std::runtime_error(std::string("no usable sm_100a GPU: ") + mpsg_create_error());
  }
  ~Context() { mpsg_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  mpsg_ctx* get() const { return ctx_; }
  void check(int rc) const { detail::raise(ctx_, rc); }

  // Process-wide default context on device 0 (like the reference's implicit
  // host execution); one host thread at a time, like mpsg_ctx.
  static Context& instance() {
    static Context c(0);
    return c;
  }

 private:
  mpsg_ctx* ctx_ = nullptr;
};

// Accumulation order.  Lane4 / Scalar are the reference's lanes-on /
// lanes-off orders (bit-exact); Fast reorders long rows and fuses each
// product-accumulate (one renormalisation per nonzero) for throughput, and is
// checked against |y - y_ref| <= 4 * rowlen * u * sum|a||x|.
enum class Order : int { Scalar = MPSG_ORDER_SCALAR, Lane4 = MPSG_ORDER_LANE4, Fast = MPSG_ORDER_FAST };
inline Order order_of(const KernelMode& m) { return m.lanes_enabled ? Order::Lane4 : Order::Scalar; }

// ------------------------------------------------------------- matrices
// Device copy of a CsrMatrix<E> or ComplexSparseMatrix<E> (one shared
// structure) for vectors of F; with_transpose also uploads A^T for sptmv.
template <class E, class F = E>
class DeviceCsr {
  static_assert(detail::device_pair<E, F>::value,
                "mps::gpu: the device runs MultiComponent<K> x MultiComponent<K> (Pure) and "
                "double x MultiComponent<K> (Mixed) products");

 public:
  static constexpr int K = detail::mc_width<F>::value;
  static constexpr bool kMixed = std::is_same<E, double>::value;
  static constexpr int kPlanes = kMixed ? 1 : K;

  DeviceCsr(const CsrMatrix<E>& A, bool with_transpose = false, Context& ctx = Context::instance()) : ctx_(&ctx) {
    const double* planes[kPlanes];
    detail::planes_of(A, planes);
    upload(A, 0, planes, with_transpose);
  }
  DeviceCsr(const ComplexSparseMatrix<E>& A, bool with_transpose = false, Context& ctx = Context::instance())
      : ctx_(&ctx) {
    check_split_structure(A);  // sparse.hpp:254-259
    const double* planes[2 * kPlanes];
    detail::planes_of(A.re, planes);
    detail::planes_of(A.im, planes + kPlanes);
    upload(A.re, MPSG_CSR_COMPLEX, planes, with_transpose);
  }
  ~DeviceCsr() { mpsg_csr_destroy(h_); }
  DeviceCsr(const DeviceCsr&) = delete;
  DeviceCsr& operator=(const DeviceCsr&) = delete;

  std::int64_t rows() const { return nrows_; }
  std::int64_t cols() const { return ncols_; }
  bool has_transpose() const { return trans_; }
  const mpsg_csr* get() const { return h_; }
  Context& context() const { return *ctx_; }

 private:
  void upload(const CsrMatrix<E>& S, int flags, const double* const* planes, bool with_transpose) {
    flags |= (kMixed ? MPSG_CSR_MIXED : 0) | (with_transpose ? MPSG_CSR_TRANSPOSE : 0);
    ctx_->check(mpsg_csr_upload_ex(ctx_->get(), K, flags, S.nrows, S.ncols, S.indptr.data(), S.indices.data(),
                                   planes, &h_));
    nrows_ = S.nrows;
    ncols_ = S.ncols;
    trans_ = with_transpose;
  }
  Context* ctx_;
  mpsg_csr* h_ = nullptr;
  std::int64_t nrows_ = 0, ncols_ = 0;
  bool trans_ = false;
};

template <class E, class F>
std::vector<F> spmv(const DeviceCsr<E, F>& A, const std::vector<F>& v, Order order) {
  static_assert(sizeof(F) == sizeof(double) * detail::mc_width<F>::value, "MultiComponent must be K doubles");
  std::vector<F> y(static_cast<std::size_t>(A.rows()));
  A.context().check(mpsg_spmv(A.context().get(), A.get(), static_cast<int>(order), static_cast<std::int64_t>(v.size()),
                              reinterpret_cast<const double*>(v.data()), reinterpret_cast<double*>(y.data())));
  return y;
}
template <class E, class F>
std::vector<F> spmv(const DeviceCsr<E, F>& A, const std::vector<F>& v, const KernelMode& mode) {
  return spmv(A, v, order_of(mode));
}

// threads: the reference sptmv's OpenMP thread count, whose per-thread
// accumulators are merged in thread order (kernels.hpp:368-394) -- reproduced
template <class E, class F>
std::vector<F> sptmv(const DeviceCsr<E, F>& A, const std::vector<F>& v, Order order, int threads = 1) {
  std::vector<F> y(static_cast<std::size_t>(A.cols()));
  A.context().check(mpsg_sptmv_ex(A.context().get(), A.get(), static_cast<int>(order), threads,
                                  static_cast<std::int64_t>(v.size()), reinterpret_cast<const double*>(v.data()),
                                  reinterpret_cast<double*>(y.data())));
  return y;
}
template <class E, class F>
std::vector<F> sptmv(const DeviceCsr<E, F>& A, const std::vector<F>& v, const KernelMode& mode) {
  return sptmv(A, v, order_of(mode), std::max(1, mode.threads));
}

template <class E, class F>
ComplexVector<F> spmv_complex(const DeviceCsr<E, F>& A, const ComplexVector<F>& v, Order order) {
  if (v.re.size() != v.im.size()) throw std::invalid_argument("spmv_complex: re/im vector length mismatch");
  ComplexVector<F> y;
  y.re.resize(static_cast<std::size_t>(A.rows()));
  y.im.resize(static_cast<std::size_t>(A.rows()));
  A.context().check(mpsg_spmv_complex(A.context().get(), A.get(), static_cast<int>(order),
                                      static_cast<std::int64_t>(v.re.size()),
                                      reinterpret_cast<const double*>(v.re.data()),
                                      reinterpret_cast<const double*>(v.im.data()),
                                      reinterpret_cast<double*>(y.re.data()),
                                      reinterpret_cast<double*>(y.im.data())));
  return y;
}
template <class E, class F>
ComplexVector<F> spmv_complex(const DeviceCsr<E, F>& A, const ComplexVector<F>& v, const KernelMode& mode) {
  return spmv_complex(A, v, order_of(mode));
}

template <class E, class F>
ComplexVector<F> sptmv_complex(const DeviceCsr<E, F>& A, const ComplexVector<F>& v, Order order,
                               bool conjugate = false, int threads = 1) {
  if (v.re.size() != v.im.size()) throw std::invalid_argument("sptmv_complex: re/im vector length mismatch");
  ComplexVector<F> y;
  y.re.resize(static_cast<std::size_t>(A.cols()));
  y.im.resize(static_cast<std::size_t>(A.cols()));
  A.context().check(mpsg_sptmv_complex_ex(A.context().get(), A.get(), static_cast<int>(order), threads,
                                          conjugate ? 1 : 0, static_cast<std::int64_t>(v.re.size()),
                                       reinterpret_cast<const double*>(v.re.data()),
                                       reinterpret_cast<const double*>(v.im.data()),
                                       reinterpret_cast<double*>(y.re.data()),
                                       reinterpret_cast<double*>(y.im.data())));
  return y;
}

// --------------------------------------------------- upload cache (drop-in)
namespace detail {
constexpr std::size_t kCacheEntries = 8;
struct CacheKey {
  const void* addr;
  const void* indptr;
  const void* plane0;
  std::int64_t nnz, nrows, ncols;
  std::uint64_t fp;  // content fingerprint (fingerprint() below)
  bool operator<(const CacheKey& o) const {
    return std::tie(addr, indptr, plane0, nnz, nrows, ncols, fp) <
           std::tie(o.addr, o.indptr, o.plane0, o.nnz, o.nrows, o.ncols, o.fp);
  }
};
// FNV-1a over up to 1024 evenly spaced elements of an array plus its last one
// (O(1) in the matrix size: a cache hit must stay cheap next to the SpMV).
template <class T>
void fnv_sample(std::uint64_t& h, const T* p, std::int64_t n) {
  if (n <= 0 || !p) return;
  const std::int64_t step = n > 1024 ? n / 1024 : 1;
  auto mix = [&](const T& v) {
    unsigned char b[sizeof(T)];
    std::memcpy(b, &v, sizeof(T));
    for (unsigned char c : b) h = (h ^ c) * 1099511628211ull;
  };
  for (std::int64_t i = 0; i < n; i += step) mix(p[i]);
  mix(p[n - 1]);
}
template <class E>
std::uint64_t fingerprint(const CsrMatrix<E>& A) {
  std::uint64_t h = 1469598103934665603ull;
  fnv_sample(h, A.indptr.data(), static_cast<std::int64_t>(A.indptr.size()));
  fnv_sample(h, A.indices.data(), static_cast<std::int64_t>(A.indices.size()));
  const double* p[16];
  planes_of(A, p);
  for (int j = 0; j < nplanes(&A); ++j) fnv_sample(h, p[j], A.nnz());
  return h;
}
template <class E, class F>
struct CacheEntry {
  std::shared_ptr<DeviceCsr<E, F>> dev;
  std::uint64_t last_use;
};
template <class E, class F>
std::map<CacheKey, CacheEntry<E, F>>& cache() {
  static std::map<CacheKey, CacheEntry<E, F>> c;
  return c;
}
inline std::uint64_t& use_clock() {
  static std::uint64_t t = 0;
  return t;
}
template <class E>
CacheKey key_of(const CsrMatrix<E>& A) {
  const double* p[16];
  planes_of(A, p);
  return {&A, A.indptr.data(), p[0], A.nnz(), A.nrows, A.ncols, fingerprint(A)};
}
template <class E>
CacheKey key_of(const ComplexSparseMatrix<E>& A) {
  const double* p[16];
  planes_of(A.re, p);
  const std::uint64_t fp = fingerprint(A.re) * 31u + fingerprint(A.im);
  return {&A, A.re.indptr.data(), p[0], A.re.nnz(), A.re.nrows, A.re.ncols, fp};
}
template <class E, class F, class M>
const DeviceCsr<E, F>& cached(const M& A, bool need_transpose) {
  auto& c = cache<E, F>();
  const CacheKey k = key_of(A);
  auto it = c.find(k);
  if (it == c.end() || (need_transpose && !it->second.dev->has_transpose())) {
    // drop stale entries for the same address (rebuilt matrix / no transpose yet)
    for (auto jt = c.begin(); jt != c.end();) jt = (jt->first.addr == k.addr) ? c.erase(jt) : std::next(jt);
    while (c.size() >= kCacheEntries) {  // evict the least recently used
      auto lru = c.begin();
      for (auto jt = c.begin(); jt != c.end(); ++jt)
        if (jt->second.last_use < lru->second.last_use) lru = jt;
      c.erase(lru);
    }
    it = c.emplace(k, CacheEntry<E, F>{std::make_shared<DeviceCsr<E, F>>(A, need_transpose), 0}).first;
  }
  it->second.last_use = ++use_clock();
  return *it->second.dev;
}
template <class M>
void invalidate_addr(const M& A) {
  auto drop = [&](auto& c) {
    for (auto it = c.begin(); it != c.end();) it = (it->first.addr == &A) ? c.erase(it) : std::next(it);
  };
  drop(cache<MultiComponent<2>, MultiComponent<2>>());
  drop(cache<MultiComponent<3>, MultiComponent<3>>());
  drop(cache<MultiComponent<4>, MultiComponent<4>>());
  drop(cache<double, MultiComponent<2>>());
  drop(cache<double, MultiComponent<3>>());
  drop(cache<double, MultiComponent<4>>());
}
}  // namespace detail

template <class E>
void invalidate(const CsrMatrix<E>& A) {
  detail::invalidate_addr(A);
}
template <class E>
void invalidate(const ComplexSparseMatrix<E>& A) {
  detail::invalidate_addr(A);
}

// ---------------------------------------- reference-signature drop-ins
// mps::spmv (kernels.hpp:348-366)
template <class E, class F>
std::vector<F> spmv(const CsrMatrix<E>& A, const std::vector<F>& v, const KernelMode& mode) {
  if (static_cast<std::size_t>(A.ncols) != v.size()) throw std::invalid_argument(detail::dim_msg("spmv", v.size(), A.ncols));
  return spmv(detail::cached<E, F>(A, false), v, mode);
}

// mps::sptmv (kernels.hpp:368-394), the reference's one-thread order
template <class E, class F>
std::vector<F> sptmv(const CsrMatrix<E>& A, const std::vector<F>& v, const KernelMode& mode) {
  if (static_cast<std::size_t>(A.nrows) != v.size()) throw std::invalid_argument(detail::dim_msg("sptmv", v.size(), A.nrows));
  return sptmv(detail::cached<E, F>(A, true), v, mode);
}

// mps::spmv_complex (kernels.hpp:399-416)
template <class E, class F>
ComplexVector<F> spmv_complex(const ComplexSparseMatrix<E>& A, const ComplexVector<F>& v, const KernelMode& mode) {
  if (v.re.size() != v.im.size()) throw std::invalid_argument("spmv_complex: re/im vector length mismatch");
  if (static_cast<std::size_t>(A.re.ncols) != v.re.size())
    throw std::invalid_argument(detail::dim_msg("spmv", v.re.size(), A.re.ncols));
  return spmv_complex(detail::cached<E, F>(A, false), v, mode);
}

// mps::sptmv_complex (kernels.hpp:419-441); conjugate = the adjoint
template <class E, class F>
ComplexVector<F> sptmv_complex(const ComplexSparseMatrix<E>& A, const ComplexVector<F>& v, const KernelMode& mode,
                               bool conjugate = false) {
  if (v.re.size() != v.im.size()) throw std::invalid_argument("sptmv_complex: re/im vector length mismatch");
  if (static_cast<std::size_t>(A.re.nrows) != v.re.size())
    throw std::invalid_argument(detail::dim_msg("sptmv", v.re.size(), A.re.nrows));
  return sptmv_complex(detail::cached<E, F>(A, true), v, order_of(mode), conjugate, std::max(1, mode.threads));
}

// nnz-balanced contiguous row bounds (kernels.hpp:63-80)
inline std::vector<std::int64_t> partition_rows(const std::vector<std::int64_t>& indptr, std::int64_t nrows,
                                                int parts) {
  std::vector<std::int64_t> b(static_cast<std::size_t>(parts) + 1);
  if (mpsg_partition_rows(indptr.data(), nrows, parts, b.data()) != MPSG_OK)
    throw std::invalid_argument("partition_rows: bad arguments");
  return b;
}

// ------------------------------------------------------------- solvers
// The Op concept of krylov.hpp:101-120 over a device-resident matrix: the
// reference's own solve_cg / solve_bicg / ... run unchanged with it, every
// apply() being one device SpMV and every apply_transposed() one device
// SpTMV (the matrix must then be uploaded with_transpose).
template <class MatE, class VecE = MatE>
struct GpuCsrOperator {
  const DeviceCsr<MatE, VecE>* matrix = nullptr;
  int threads = 1;  // apply_transposed / BiCG: the reference sptmv's per-thread merge order
  bool lanes_enabled = true;
  bool fast = false;

  std::int64_t rows() const { return matrix->rows(); }
  std::int64_t cols() const { return matrix->cols(); }
  KernelMode mode() const { return KernelMode{{}, MatrixMode::Pure, false, threads, lanes_enabled}; }
  Order order() const { return fast ? Order::Fast : order_of(mode()); }
  template <class F>
  std::vector<F> apply(const std::vector<F>& x) const {
    return gpu::spmv(*matrix, x, order());
  }
  template <class F>
  std::vector<F> apply_transposed(const std::vector<F>& x) const {
    return gpu::sptmv(*matrix, x, order(), threads);  // the reference's thread-count-dependent merge
  }
};

namespace detail {
template <class MatE, class E>
void check_solve_args(const GpuCsrOperator<MatE, E>& op, const std::vector<E>& b, const SolverConfig& cfg,
                      std::vector<E>& x0) {
  cfg.validate();  // krylov.hpp:69-75
  if (op.rows() != op.cols())
    throw std::invalid_argument("solver: operator must be square, got " + std::to_string(op.rows()) + "x" +
                                std::to_string(op.cols()));
  if (static_cast<std::size_t>(op.cols()) != b.size())
    throw std::invalid_argument("solver: rhs length does not match the operator");
  if (!cfg.x0.empty()) {
    if (cfg.x0.size() != b.size()) throw std::invalid_argument("solver: x0 length does not match the rhs");
    x0.resize(b.size());
    for (std::size_t i = 0; i < b.size(); ++i) x0[i] = E(cfg.x0[i]);  // scalar_like (krylov.hpp:178)
  }
}
template <class MatE, class E>
int solve_order(const GpuCsrOperator<MatE, E>& op, const SolverConfig& cfg) {
  return op.fast ? MPSG_ORDER_FAST : (cfg.lanes_enabled && op.lanes_enabled ? MPSG_ORDER_LANE4 : MPSG_ORDER_SCALAR);
}
template <class E>
void fill_report(SolverReport& r, const mpsg_cg_report& rep, const std::vector<double>& hist) {
  r.status = static_cast<SolverStatus>(rep.status);
  r.converged = rep.converged != 0;
  r.detail = rep.detail;
  r.iterations = rep.iterations;
  r.residual_history.assign(hist.begin(), hist.begin() + rep.history_len);
  r.rhs_norm = rep.rhs_norm;
  r.final_recurrence_residual = rep.final_recurrence_residual;
  r.final_true_residual = rep.final_true_residual;
  r.setup_seconds = rep.setup_seconds;
  r.solve_seconds = rep.solve_seconds;
}
}  // namespace detail

// Device-resident CG (krylov.hpp:238-281): vectors and scalars never leave
// the GPU; the residual history, status and true residual come back in the
// reference's SolverReport.  Only rel_tol, abs_tol, max_iters, x0 and
// lanes_enabled of SolverConfig are read (as by the reference CG).  Pure or
// Mixed mode (GpuCsrOperator<double, MultiComponent<K>>, as CsrOperator<double>
// with a multi-component rhs in the reference's solve_core, bench.cpp:550-557).
template <class MatE, class E>
SolveResult<E> solve_cg(const GpuCsrOperator<MatE, E>& op, const std::vector<E>& b, const SolverConfig& cfg) {
  constexpr int K = detail::mc_width<E>::value;
  static_assert(K >= 2, "device CG runs on MultiComponent<K>");
  std::vector<E> x0;
  detail::check_solve_args(op, b, cfg, x0);
  mpsg_cg_config c{cfg.rel_tol, cfg.abs_tol, cfg.max_iters, 32, 1};
  mpsg_cg_report rep{};
  SolveResult<E> res;
  res.x.resize(b.size());
  std::vector<double> hist(static_cast<std::size_t>(cfg.max_iters) + 1);
  Context& ctx = op.matrix->context();
  ctx.check(mpsg_cg(ctx.get(), op.matrix->get(), detail::solve_order(op, cfg), static_cast<std::int64_t>(b.size()),
                    reinterpret_cast<const double*>(b.data()),
                    x0.empty() ? nullptr : reinterpret_cast<const double*>(x0.data()), &c,
                    reinterpret_cast<double*>(res.x.data()), hist.data(), static_cast<std::int64_t>(hist.size()),
                    &rep));
  detail::fill_report<E>(res.report, rep, hist);
  return res;
}

// Dot-product order of the device solvers: Tree (throughput; deterministic,
// not the reference's bits) or Sequential (the reference's serial dot,
// krylov.hpp:122-128 -- with lanes on/off this reproduces the reference
// solver bit for bit: iterate, history, status, detail).
enum class DotOrder { Tree = MPSG_DOT_TREE, Sequential = MPSG_DOT_SEQUENTIAL };

// Device-resident solve() (krylov.hpp:596-606) and the per-method entry
// points (solve_bicg :283, solve_cgs :339, solve_bicgstab :398, solve_gpbicg
// :478).  Reads method, rel_tol, abs_tol, max_iters, x0, lanes_enabled of
// SolverConfig; BiCG's transposed products follow the operator's thread count
// (the reference's per-thread merge) and need a DeviceCsr uploaded with the
// transpose.  Real, Pure or Mixed mode.
template <class MatE, class E>
SolveResult<E> solve_method(const GpuCsrOperator<MatE, E>& op, const std::vector<E>& b, const SolverConfig& cfg,
                            KrylovMethod method, DotOrder dots = DotOrder::Tree) {
  constexpr int K = detail::mc_width<E>::value;
  static_assert(K >= 2, "device solvers run on MultiComponent<K>");
  std::vector<E> x0;
  detail::check_solve_args(op, b, cfg, x0);
  mpsg_solver_config c{};
  c.method = static_cast<int32_t>(method);
  c.threads = std::max(op.threads, 1);
  c.rel_tol = cfg.rel_tol;
  c.abs_tol = cfg.abs_tol;
  c.max_iters = cfg.max_iters;
  c.check_every = 32;
  c.use_graph = 1;
  c.dot_order = static_cast<int32_t>(dots);
  mpsg_cg_report rep{};
  SolveResult<E> res;
  res.x.resize(b.size());
  std::vector<double> hist(static_cast<std::size_t>(cfg.max_iters) + 1);
  Context& ctx = op.matrix->context();
  ctx.check(mpsg_solve(ctx.get(), op.matrix->get(), detail::solve_order(op, cfg), static_cast<std::int64_t>(b.size()),
                       reinterpret_cast<const double*>(b.data()),
                       x0.empty() ? nullptr : reinterpret_cast<const double*>(x0.data()), &c,
                       reinterpret_cast<double*>(res.x.data()), hist.data(), static_cast<std::int64_t>(hist.size()),
                       &rep));
  detail::fill_report<E>(res.report, rep, hist);
  return res;
}
template <class MatE, class E>
SolveResult<E> solve(const GpuCsrOperator<MatE, E>& op, const std::vector<E>& b, const SolverConfig& cfg,
                     DotOrder dots = DotOrder::Tree) {
  return solve_method(op, b, cfg, cfg.method, dots);
}
template <class MatE, class E>
SolveResult<E> solve_bicg(const GpuCsrOperator<MatE, E>& op, const std::vector<E>& b, const SolverConfig& cfg,
                          DotOrder dots = DotOrder::Tree) {
  return solve_method(op, b, cfg, KrylovMethod::BiCG, dots);
}
template <class MatE, class E>
SolveResult<E> solve_cgs(const GpuCsrOperator<MatE, E>& op, const std::vector<E>& b, const SolverConfig& cfg,
                         DotOrder dots = DotOrder::Tree) {
  return solve_method(op, b, cfg, KrylovMethod::CGS, dots);
}
template <class MatE, class E>
SolveResult<E> solve_bicgstab(const GpuCsrOperator<MatE, E>& op, const std::vector<E>& b, const SolverConfig& cfg,
                              DotOrder dots = DotOrder::Tree) {
  return solve_method(op, b, cfg, KrylovMethod::BiCGSTAB, dots);
}
template <class MatE, class E>
SolveResult<E> solve_gpbicg(const GpuCsrOperator<MatE, E>& op, const std::vector<E>& b, const SolverConfig& cfg,
                            DotOrder dots = DotOrder::Tree) {
  return solve_method(op, b, cfg, KrylovMethod::GPBiCG, dots);
}

}  // namespace gpu
}  // namespace mps
