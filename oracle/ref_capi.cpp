// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY: a C-ABI shim over the UNMODIFIED
// reference library, compiled straight from /root/reference/proj/include by
// oracle/Makefile into oracle/_ref/libmpsref.so (git-ignored; it travels to
// the GPU box with the snapshot).  Nothing in the product links this file.
//
// It exposes the reference's own entry points -- mps::spmv (kernels.hpp:348),
// mps::spmv_complex (kernels.hpp:399), mps::solve_cg (krylov.hpp:238), the
// MultiComponent ops (multicomp.hpp:225-322), make_vector / checksum
// (bench.hpp:78-150) and the test fixtures (tests/support/fixtures.hpp) -- so
// the Python tests can pin the C restatement (oracle/mpsoracle.c) and the
// CUDA path against the reference bit-for-bit, and bench.py can time the
// reference CPU path (`--impl reference`, cpu_baseline).
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "mps/bench.hpp"
#include "mps/mtxio.hpp"
#include "mps/kernels.hpp"
#include "mps/krylov.hpp"
#include "support/fixtures.hpp"

using namespace mps;

namespace {

thread_local std::string g_err;

template <int K>
using MC = MultiComponent<K>;

using AnyCsr = std::variant<CsrMatrix<double>, CsrMatrix<MC<2>>, CsrMatrix<MC<3>>, CsrMatrix<MC<4>>>;
using AnyVec = std::variant<std::vector<MC<2>>, std::vector<MC<3>>, std::vector<MC<4>>>;

struct CsrH {
  int K;  // 1 = binary64 matrix (mixed mode)
  AnyCsr m;
};
struct ComplexH {
  int K;  // 1 = binary64 matrix (mixed mode)
  std::variant<ComplexSparseMatrix<MC<2>>, ComplexSparseMatrix<MC<3>>, ComplexSparseMatrix<MC<4>>,
               ComplexSparseMatrix<double>>
      m;
};
struct VecH {
  int K;
  AnyVec v;
};
struct CVecH {
  int K;
  std::variant<ComplexVector<MC<2>>, ComplexVector<MC<3>>, ComplexVector<MC<4>>> v;
};

template <class E>
CsrMatrix<E> build_csr(int64_t nrows, int64_t ncols, const int64_t* indptr, const int64_t* indices,
                       const double* vals) {
  CsrMatrix<E> m;
  m.nrows = nrows;
  m.ncols = ncols;
  int64_t nnz = indptr[nrows];
  m.indptr.assign(indptr, indptr + nrows + 1);
  m.indices.assign(indices, indices + nnz);
  m.values.resize(static_cast<size_t>(nnz));
  for (int64_t k = 0; k < nnz; ++k) {
    if constexpr (std::is_same_v<E, double>) {
      m.values.set(static_cast<size_t>(k), vals[k]);
    } else {
      E e;
      for (size_t j = 0; j < e.c.size(); ++j) e.c[j] = vals[static_cast<int64_t>(j) * nnz + k];
      m.values.set(static_cast<size_t>(k), e);
    }
  }
  return m;
}

template <int K>
std::vector<MC<K>> build_vec(int64_t n, const double* aos) {
  std::vector<MC<K>> v(static_cast<size_t>(n));
  if (n) std::memcpy(v.data(), aos, static_cast<size_t>(n) * K * sizeof(double));
  return v;
}

template <int K>
void read_vec(const std::vector<MC<K>>& v, double* aos) {
  if (!v.empty()) std::memcpy(aos, v.data(), v.size() * K * sizeof(double));
}

template <class Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

KernelMode mode_of(int lanes, int threads) {
  KernelMode m;
  m.threads = threads;
  m.lanes_enabled = lanes != 0;
  return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- matrices / vectors ------------------------------------------------
void* ref_csr_create(int K, int64_t nrows, int64_t ncols, const int64_t* indptr,
                     const int64_t* indices, const double* vals) {
  auto* h = new CsrH{K, CsrMatrix<double>{}};
  switch (K) {
    case 1: h->m = build_csr<double>(nrows, ncols, indptr, indices, vals); break;
    case 2: h->m = build_csr<MC<2>>(nrows, ncols, indptr, indices, vals); break;
    case 3: h->m = build_csr<MC<3>>(nrows, ncols, indptr, indices, vals); break;
    case 4: h->m = build_csr<MC<4>>(nrows, ncols, indptr, indices, vals); break;
    default: delete h; return nullptr;
  }
  return h;
}
void ref_csr_destroy(void* h) { delete static_cast<CsrH*>(h); }

void* ref_vec_create(int K, int64_t n, const double* aos) {
  auto* h = new VecH{K, std::vector<MC<2>>{}};
  switch (K) {
    case 2: h->v = build_vec<2>(n, aos); break;
    case 3: h->v = build_vec<3>(n, aos); break;
    case 4: h->v = build_vec<4>(n, aos); break;
    default: delete h; return nullptr;
  }
  return h;
}
void ref_vec_destroy(void* h) { delete static_cast<VecH*>(h); }
int64_t ref_vec_size(void* h) {
  return std::visit([](auto& v) { return static_cast<int64_t>(v.size()); }, static_cast<VecH*>(h)->v);
}
void ref_vec_read(void* h, double* aos) {
  std::visit([&](auto& v) { read_vec(v, aos); }, static_cast<VecH*>(h)->v);
}
uint64_t ref_vec_checksum(void* h) {
  return std::visit([](auto& v) { return checksum(v); }, static_cast<VecH*>(h)->v);
}

// mps::spmv (kernels.hpp:348-366).  `out` receives the returned vector.
// Pure mode when the matrix has the vector's K; mixed mode for a binary64
// matrix (K == 1).  Timing callers measure exactly this call.
int ref_spmv(void* A, void* v, int lanes, int threads, void* out) {
  auto* a = static_cast<CsrH*>(A);
  auto* x = static_cast<VecH*>(v);
  auto* y = static_cast<VecH*>(out);
  KernelMode mode = mode_of(lanes, threads);
  return guard([&] {
    std::visit(
        [&](auto& mat, auto& vec) {
          using MatT = std::decay_t<decltype(mat)>;
          using VecT = std::decay_t<decltype(vec)>;
          using E = std::decay_t<decltype(mat.values.get(0))>;
          using F = typename VecT::value_type;
          if constexpr (std::is_same_v<E, F> || std::is_same_v<E, double>) {
            (void)sizeof(MatT);
            y->v = spmv(mat, vec, mode);
            y->K = x->K;
          } else {
            throw std::runtime_error("ref_spmv: matrix/vector precision mismatch");
          }
        },
        a->m, x->v);
  });
}

// mps::sptmv (kernels.hpp:368-394), for the transposed-product pins.
int ref_sptmv(void* A, void* v, int lanes, int threads, void* out) {
  auto* a = static_cast<CsrH*>(A);
  auto* x = static_cast<VecH*>(v);
  auto* y = static_cast<VecH*>(out);
  KernelMode mode = mode_of(lanes, threads);
  return guard([&] {
    std::visit(
        [&](auto& mat, auto& vec) {
          using VecT = std::decay_t<decltype(vec)>;
          using E = std::decay_t<decltype(mat.values.get(0))>;
          using F = typename VecT::value_type;
          if constexpr (std::is_same_v<E, F> || std::is_same_v<E, double>) {
            y->v = sptmv(mat, vec, mode);
            y->K = x->K;
          } else {
            throw std::runtime_error("ref_sptmv: matrix/vector precision mismatch");
          }
        },
        a->m, x->v);
  });
}

// ---- complex -----------------------------------------------------------
void* ref_ccsr_create(int K, int64_t nrows, int64_t ncols, const int64_t* indptr,
                      const int64_t* indices, const double* re_vals, const double* im_vals) {
  auto* h = new ComplexH{K, ComplexSparseMatrix<MC<2>>{}};
  switch (K) {
    case 1:
      h->m = ComplexSparseMatrix<double>{build_csr<double>(nrows, ncols, indptr, indices, re_vals),
                                         build_csr<double>(nrows, ncols, indptr, indices, im_vals)};
      break;
    case 2:
      h->m = ComplexSparseMatrix<MC<2>>{build_csr<MC<2>>(nrows, ncols, indptr, indices, re_vals),
                                        build_csr<MC<2>>(nrows, ncols, indptr, indices, im_vals)};
      break;
    case 3:
      h->m = ComplexSparseMatrix<MC<3>>{build_csr<MC<3>>(nrows, ncols, indptr, indices, re_vals),
                                        build_csr<MC<3>>(nrows, ncols, indptr, indices, im_vals)};
      break;
    case 4:
      h->m = ComplexSparseMatrix<MC<4>>{build_csr<MC<4>>(nrows, ncols, indptr, indices, re_vals),
                                        build_csr<MC<4>>(nrows, ncols, indptr, indices, im_vals)};
      break;
    default: delete h; return nullptr;
  }
  return h;
}
void ref_ccsr_destroy(void* h) { delete static_cast<ComplexH*>(h); }

void* ref_cvec_create(int K, int64_t n, const double* re, const double* im) {
  auto* h = new CVecH{K, ComplexVector<MC<2>>{}};
  switch (K) {
    case 2: h->v = ComplexVector<MC<2>>{build_vec<2>(n, re), build_vec<2>(n, im)}; break;
    case 3: h->v = ComplexVector<MC<3>>{build_vec<3>(n, re), build_vec<3>(n, im)}; break;
    case 4: h->v = ComplexVector<MC<4>>{build_vec<4>(n, re), build_vec<4>(n, im)}; break;
    default: delete h; return nullptr;
  }
  return h;
}
void ref_cvec_destroy(void* h) { delete static_cast<CVecH*>(h); }
void ref_cvec_read(void* h, double* re, double* im) {
  std::visit([&](auto& v) { read_vec(v.re, re); read_vec(v.im, im); }, static_cast<CVecH*>(h)->v);
}
uint64_t ref_cvec_checksum(void* h) {
  return std::visit([](auto& v) { return checksum(v); }, static_cast<CVecH*>(h)->v);
}

// mps::spmv_complex (kernels.hpp:399-416)
int ref_spmv_complex(void* A, void* v, int lanes, int threads, void* out) {
  auto* a = static_cast<ComplexH*>(A);
  auto* x = static_cast<CVecH*>(v);
  auto* y = static_cast<CVecH*>(out);
  KernelMode mode = mode_of(lanes, threads);
  return guard([&] {
    std::visit(
        [&](auto& mat, auto& vec) {
          using E = std::decay_t<decltype(mat.re.values.get(0))>;
          using F = typename decltype(vec.re)::value_type;
          if constexpr (std::is_same_v<E, F> || std::is_same_v<E, double>) {
            y->v = spmv_complex(mat, vec, mode);
            y->K = x->K;
          } else {
            throw std::runtime_error("ref_spmv_complex: precision mismatch");
          }
        },
        a->m, x->v);
  });
}

// mps::sptmv_complex (kernels.hpp:419-441), conjugate = adjoint
int ref_sptmv_complex(void* A, void* v, int lanes, int threads, int conjugate, void* out) {
  auto* a = static_cast<ComplexH*>(A);
  auto* x = static_cast<CVecH*>(v);
  auto* y = static_cast<CVecH*>(out);
  KernelMode mode = mode_of(lanes, threads);
  return guard([&] {
    std::visit(
        [&](auto& mat, auto& vec) {
          using E = std::decay_t<decltype(mat.re.values.get(0))>;
          using F = typename decltype(vec.re)::value_type;
          if constexpr (std::is_same_v<E, F> || std::is_same_v<E, double>) {
            y->v = sptmv_complex(mat, vec, mode, conjugate != 0);
            y->K = x->K;
          } else {
            throw std::runtime_error("ref_sptmv_complex: precision mismatch");
          }
        },
        a->m, x->v);
  });
}

// ---- scalar multi-component ops (multicomp.hpp:225-335) -----------------
// op: 0 add, 1 mul, 2 mul_by_double(a, b[0]), 3 sub, 4 divide, 5 sqrt(a)
void ref_mc_op(int op, int K, const double* a, const double* b, double* out) {
  auto run = [&](auto proto) {
    using E = decltype(proto);
    E x, y, r;
    for (size_t j = 0; j < x.c.size(); ++j) {
      x.c[j] = a[j];
      y.c[j] = b[j];
    }
    switch (op) {
      case 0: r = add(x, y); break;
      case 1: r = mul(x, y); break;
      case 2: r = mul_by_double(x, b[0]); break;
      case 3: r = sub(x, y); break;
      case 4: r = divide(x, y); break;
      case 5: r = mps::sqrt(x); break;
      default: break;
    }
    for (size_t j = 0; j < r.c.size(); ++j) out[j] = r.c[j];
  };
  if (K == 2) run(MC<2>{});
  if (K == 3) run(MC<3>{});
  if (K == 4) run(MC<4>{});
}

// ---- make_vector (bench.hpp:78-111) -------------------------------------
void ref_make_vector(int K, int64_t n, double* out) {
  if (K == 2) read_vec(make_vector<MC<2>>(n, MC<2>{}), out);
  if (K == 3) read_vec(make_vector<MC<3>>(n, MC<3>{}), out);
  if (K == 4) read_vec(make_vector<MC<4>>(n, MC<4>{}), out);
}
void ref_make_complex_vector(int K, int64_t n, double* re, double* im) {
  auto go = [&](auto proto) {
    auto v = make_complex_vector(n, proto);
    read_vec(v.re, re);
    read_vec(v.im, im);
  };
  if (K == 2) go(MC<2>{});
  if (K == 3) go(MC<3>{});
  if (K == 4) go(MC<4>{});
}

// ---- solve_cg (krylov.hpp:238-281) through the reference CsrOperator ------
// Returns the number of history entries written (or -1 on an exception).
int64_t ref_cg(void* A, void* b, int lanes, int threads, double rel_tol, double abs_tol,
               int64_t max_iters, double* x_out, double* history, int64_t hist_cap,
               int64_t* iterations, int* status, double* rhs_norm, double* final_true,
               double* final_rec, char* detail, int detail_cap) {
  auto* a = static_cast<CsrH*>(A);
  auto* bv = static_cast<VecH*>(b);
  int64_t written = -1;
  int rc = guard([&] {
    std::visit(
        [&](auto& mat, auto& vec) {
          using E = std::decay_t<decltype(mat.values.get(0))>;
          using F = typename std::decay_t<decltype(vec)>::value_type;
          // Pure (E == F) or Mixed (E = double: CsrOperator<double>, bench.cpp:550-557)
          if constexpr (std::is_same_v<E, F> || (std::is_same_v<E, double> && !std::is_same_v<F, double>)) {
            CsrOperator<E> op{&mat, threads, lanes != 0};
            SolverConfig cfg;
            cfg.method = KrylovMethod::CG;
            cfg.rel_tol = rel_tol;
            cfg.abs_tol = abs_tol;
            cfg.max_iters = max_iters;
            cfg.threads = threads;
            cfg.lanes_enabled = lanes != 0;
            auto res = solve_cg(op, vec, cfg);
            read_vec(res.x, x_out);
            int64_t n = static_cast<int64_t>(res.report.residual_history.size());
            written = n < hist_cap ? n : hist_cap;
            for (int64_t i = 0; i < written; ++i) history[i] = res.report.residual_history[i];
            *iterations = res.report.iterations;
            *status = static_cast<int>(res.report.status);
            *rhs_norm = res.report.rhs_norm;
            *final_true = res.report.final_true_residual;
            *final_rec = res.report.final_recurrence_residual;
            if (detail_cap > 0) {
              std::strncpy(detail, res.report.detail.c_str(), static_cast<size_t>(detail_cap - 1));
              detail[detail_cap - 1] = 0;
            }
          } else {
            throw std::runtime_error("ref_cg: precision mismatch");
          }
        },
        a->m, bv->v);
  });
  return rc == 0 ? written : -1;
}

// ---- solve() (krylov.hpp:596-606): every KrylovMethod through CsrOperator --
// method: KrylovMethod order (CG, BiCG, CGS, BiCGSTAB, GPBiCG); x0 NULL = zero.
int64_t ref_solve(void* A, void* b, int method, int lanes, int threads, double rel_tol, double abs_tol,
                  int64_t max_iters, const double* x0, double* x_out, double* history, int64_t hist_cap,
                  int64_t* iterations, int* status, double* rhs_norm, double* final_true, double* final_rec,
                  char* detail, int detail_cap) {
  auto* a = static_cast<CsrH*>(A);
  auto* bv = static_cast<VecH*>(b);
  int64_t written = -1;
  int rc = guard([&] {
    std::visit(
        [&](auto& mat, auto& vec) {
          using E = std::decay_t<decltype(mat.values.get(0))>;
          using F = typename std::decay_t<decltype(vec)>::value_type;
          // Pure (E == F) or Mixed (E = double: CsrOperator<double>, bench.cpp:550-557)
          if constexpr (std::is_same_v<E, F> || (std::is_same_v<E, double> && !std::is_same_v<F, double>)) {
            CsrOperator<E> op{&mat, threads, lanes != 0};
            SolverConfig cfg;
            cfg.method = static_cast<KrylovMethod>(method);
            cfg.rel_tol = rel_tol;
            cfg.abs_tol = abs_tol;
            cfg.max_iters = max_iters;
            cfg.threads = threads;
            cfg.lanes_enabled = lanes != 0;
            if (x0) cfg.x0.assign(x0, x0 + vec.size());
            auto res = solve(op, vec, cfg);
            read_vec(res.x, x_out);
            int64_t n = static_cast<int64_t>(res.report.residual_history.size());
            written = n < hist_cap ? n : hist_cap;
            for (int64_t i = 0; i < written; ++i) history[i] = res.report.residual_history[i];
            *iterations = res.report.iterations;
            *status = static_cast<int>(res.report.status);
            *rhs_norm = res.report.rhs_norm;
            *final_true = res.report.final_true_residual;
            *final_rec = res.report.final_recurrence_residual;
            if (detail_cap > 0) {
              std::strncpy(detail, res.report.detail.c_str(), static_cast<size_t>(detail_cap - 1));
              detail[detail_cap - 1] = 0;
            }
          } else {
            throw std::runtime_error("ref_solve: precision mismatch");
          }
        },
        a->m, bv->v);
  });
  return rc == 0 ? written : -1;
}

// ---- reference test fixtures (tests/support/fixtures.hpp) ---------------
// name: "example5x5", "tub1000", "qc324_re", "qc324_im", "random_coo" (seed,
// nrows, ncols, nnz), "diag_dominant_sym" (seed, n, density*1e6).
void* ref_fixture(const char* name, uint64_t seed, int64_t a, int64_t b, int64_t c) {
  std::string s(name);
  auto* h = new CsrH{1, CsrMatrix<double>{}};
  if (s == "example5x5") {
    CooMatrix<double> coo;
    coo.nrows = coo.ncols = 5;
    coo.entries = {{0, 0, 1.0}, {0, 2, 2.0},  {1, 1, 3.0}, {1, 4, -4.0},
                   {2, 2, 5.0}, {3, 0, 6.0}, {3, 3, -7.0}, {4, 4, 8.0}};
    h->m = coo_to_csr(coo);
  } else if (s == "tub1000") {
    h->m = coo_to_csr(test::tub1000_standin());
  } else if (s == "qc324_re" || s == "qc324_im") {
    auto cm = split_complex(test::qc324_standin());
    h->m = (s == "qc324_re") ? cm.re : cm.im;
  } else if (s == "random_coo") {
    test::Rng rng(seed);
    h->m = coo_to_csr(test::random_coo(rng, a, b, static_cast<int>(c)));
  } else if (s == "diag_dominant_sym") {
    test::Rng rng(seed);
    h->m = coo_to_csr(test::random_diag_dominant(rng, a, static_cast<double>(b) * 1e-6, true));
  } else {
    delete h;
    return nullptr;
  }
  return h;
}
void ref_csr_info(void* h, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
  std::visit(
      [&](auto& m) {
        *nrows = m.nrows;
        *ncols = m.ncols;
        *nnz = m.nnz();
      },
      static_cast<CsrH*>(h)->m);
}
// Export a binary64 matrix (K == 1 handle) as int64 CSR arrays.
int ref_csr_export(void* hh, int64_t* indptr, int64_t* indices, double* vals) {
  auto* h = static_cast<CsrH*>(hh);
  if (h->K != 1) return 1;
  auto& m = std::get<CsrMatrix<double>>(h->m);
  std::memcpy(indptr, m.indptr.data(), m.indptr.size() * sizeof(int64_t));
  std::memcpy(indices, m.indices.data(), m.indices.size() * sizeof(int64_t));
  for (int64_t k = 0; k < m.nnz(); ++k) vals[k] = m.values.get(static_cast<size_t>(k));
  return 0;
}

// The reference CLI's spmv pipeline (tools/mpsparse.cpp:74-97 -> time_kernel,
// src/bench.cpp:192-253) on a Matrix Market file: returns the record's
// checksum and fills n / nnz.  K = 2, 3, 4; mixed = binary64 matrix.
int ref_mtx_spmv(const char* path, int K, int mixed, int lanes, int threads, int transposed, uint64_t* checksum_out,
                 int64_t* n_out, int64_t* nnz_out) {
  return guard([&] {
    auto parsed = parse_mtx_file(path, true);
    KernelRequest req;
    req.precision = K == 2 ? PrecisionTag::dd() : K == 3 ? PrecisionTag::td() : PrecisionTag::qd();
    req.matrix_mode = mixed ? MatrixMode::MixedBinary64 : MatrixMode::Pure;
    req.threads = threads;
    req.lanes_enabled = lanes != 0;
    req.repetitions = 1;
    BenchRecord rec;
    if (is_complex(parsed)) {
      req.kernel = transposed ? KernelKind::SptmvComplex : KernelKind::SpmvComplex;
      rec = time_kernel(split_complex(std::get<CooMatrix<std::complex<double>>>(parsed)), "m", req);
    } else {
      req.kernel = transposed ? KernelKind::Sptmv : KernelKind::Spmv;
      rec = time_kernel(coo_to_csr(std::get<CooMatrix<double>>(parsed)), "m", req);
    }
    *checksum_out = rec.checksum;
    *n_out = rec.n;
    *nnz_out = rec.nnz;
  });
}

}  // extern "C"
