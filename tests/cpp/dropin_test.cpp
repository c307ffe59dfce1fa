// dropin_test.cpp -- the C++ drop-in (include/mps/gpu.hpp) exercised against
// the UNMODIFIED reference, compiled together from the reference headers
// (/root/reference/proj/include, tests/support) by `make -C oracle dropin`
// into oracle/_ref/dropin_test (git-ignored; travels to the GPU box).  Run by
// tests/test_gpu_dropin.py on a B200.  Each check prints PASS/FAIL; the exit
// status is the number of failures.
//
// What it pins (reference file:line):
//  1. mps::gpu::spmv == mps::spmv bit for bit, lanes on and off, K = 2, 3, 4,
//     on the 5x5 worked example (test_kernels.cpp:99-138), the tub1000
//     stand-in (fixtures.hpp:23) and random full-precision matrices;
//  2. mps::gpu::spmv_complex == mps::spmv_complex bit for bit on the qc324
//     stand-in (fixtures.hpp:125) and a random complex matrix;
//  3. the reference's own solve_cg (krylov.hpp:238) driven by a
//     GpuCsrOperator produces the same residual history, iterate and status as
//     with the host CsrOperator (the SpMV is bit-exact, everything else is the
//     reference's own code);
//  4. the device-resident mps::gpu::solve_cg tracks the reference CG on the
//     nd3k stand-in (fixtures.hpp:45) and diag(1..40);
//  5. errors: dimension mismatch throws std::invalid_argument with the
//     reference's text (kernels.hpp:333-339);
//  6. Mixed mode (CsrMatrix<double> x MultiComponent<K>, kernels.hpp:55-58)
//     and the transposed products mps::gpu::sptmv / sptmv_complex (+ adjoint)
//     bit for bit against the reference at one thread (kernels.hpp:368-441);
//  7. the reference's own solve_bicg (krylov.hpp:283, uses apply_transposed)
//     over a GpuCsrOperator: identical history to the host operator;
//  8. the device-resident mps::gpu::solve (every KrylovMethod, krylov.hpp:
//     596-606) with DotOrder::Sequential == the reference's mps::solve bit for
//     bit (iterate, history, status, iterations, detail, true residual), lanes
//     on and off, BiCG at 1 and 4 threads; with DotOrder::Tree the same status
//     within +-1 iteration.
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "mps/bench.hpp"
#include "mps/kernels.hpp"
#include "mps/krylov.hpp"
#include "mps/gpu.hpp"
#include "support/fixtures.hpp"

using namespace mps;

namespace {

int failures = 0;

std::string sci(double v) {
  char b[32];
  std::snprintf(b, sizeof(b), "%.6e", v);
  return b;
}

void report(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

template <int K>
bool same_bits(const std::vector<MultiComponent<K>>& a, const std::vector<MultiComponent<K>>& b) {
  if (a.size() != b.size()) return false;
  return a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(a[0])) == 0;
}

CsrMatrix<double> example5x5() {
  CooMatrix<double> coo;
  coo.nrows = coo.ncols = 5;
  coo.entries = {{0, 0, 1.0}, {0, 2, 2.0}, {1, 1, 3.0}, {1, 4, -4.0},
                 {2, 2, 5.0}, {3, 0, 6.0}, {3, 3, -7.0}, {4, 4, 8.0}};
  return coo_to_csr(coo);
}

// Full-precision values on a given structure (Rng::multicomp, oracle.hpp:90).
template <int K>
CsrMatrix<MultiComponent<K>> full_precision(const CsrMatrix<double>& s, test::Rng& rng) {
  auto A = convert_csr<MultiComponent<K>>(s);
  for (std::size_t i = 0; i < A.indices.size(); ++i) A.values.set(i, rng.multicomp<K>(-4, 4));
  return A;
}
template <int K>
std::vector<MultiComponent<K>> random_vector(std::int64_t n, test::Rng& rng) {
  std::vector<MultiComponent<K>> v(static_cast<std::size_t>(n));
  for (auto& e : v) e = rng.multicomp<K>(-4, 4);
  return v;
}

template <int K>
void spmv_case(const std::string& name, const CsrMatrix<MultiComponent<K>>& A,
               const std::vector<MultiComponent<K>>& v) {
  for (bool lanes : {true, false}) {
    KernelMode m{{}, MatrixMode::Pure, false, 4, lanes};
    auto ref = mps::spmv(A, v, m);
    auto got = mps::gpu::spmv(A, v, m);
    report(same_bits(ref, got) && checksum(ref) == checksum(got),
           name + " K=" + std::to_string(K) + (lanes ? " lanes on" : " lanes off") + " spmv bit-exact");
  }
}

template <int K>
void spmv_suite(test::Rng& rng) {
  auto ex = convert_csr<MultiComponent<K>>(example5x5());
  std::vector<MultiComponent<K>> v5;
  for (int i = 1; i <= 5; ++i) v5.push_back(MultiComponent<K>(double(i)));
  spmv_case<K>("example5x5", ex, v5);
  auto y = mps::gpu::spmv(ex, v5, KernelMode{});
  const double want[5] = {7, -14, 15, -22, 40};  // test_kernels.cpp:99-138
  bool exact = true;
  for (int i = 0; i < 5; ++i) exact = exact && y[i].c[0] == want[i] && y[i].c[1] == 0.0;
  report(exact, "example5x5 K=" + std::to_string(K) + " equals [7 -14 15 -22 40]");

  auto tub = full_precision<K>(coo_to_csr(test::tub1000_standin()), rng);
  spmv_case<K>("tub1000", tub, random_vector<K>(tub.ncols, rng));
  auto rnd = full_precision<K>(coo_to_csr(test::random_coo(rng, 700, 650, 24000)), rng);
  spmv_case<K>("random 700x650", rnd, random_vector<K>(rnd.ncols, rng));
  // widened binary64 values (integer-ish data takes renorm's general path)
  auto wide = convert_csr<MultiComponent<K>>(coo_to_csr(test::tub1000_standin()));
  std::vector<MultiComponent<K>> wv;
  for (std::int64_t i = 0; i < wide.ncols; ++i) wv.push_back(MultiComponent<K>(std::sqrt(2.0) * double(i)));
  spmv_case<K>("tub1000 widened", wide, wv);
}

template <int K>
void complex_suite(test::Rng& rng) {
  for (int which = 0; which < 2; ++which) {
    auto cm = which == 0 ? split_complex(test::qc324_standin())
                         : split_complex(test::random_complex_coo(rng, 300, 300, 9000));
    auto A = convert_complex_csr<MultiComponent<K>>(cm);
    for (std::size_t i = 0; i < A.re.indices.size(); ++i) {
      A.re.values.set(i, rng.multicomp<K>(-4, 4));
      A.im.values.set(i, rng.multicomp<K>(-4, 4));
    }
    ComplexVector<MultiComponent<K>> v{random_vector<K>(A.ncols(), rng), random_vector<K>(A.ncols(), rng)};
    for (bool lanes : {true, false}) {
      KernelMode m{{}, MatrixMode::Pure, false, 1, lanes};
      auto ref = mps::spmv_complex(A, v, m);
      auto got = mps::gpu::spmv_complex(A, v, m);
      report(same_bits(ref.re, got.re) && same_bits(ref.im, got.im),
             std::string(which == 0 ? "qc324" : "random complex") + " K=" + std::to_string(K) +
                 (lanes ? " lanes on" : " lanes off") + " spmv_complex bit-exact");
    }
  }
}

template <int K>
void solver_suite() {
  using E = MultiComponent<K>;
  auto A = convert_csr<E>(test::nd3k_standin());
  auto xt = make_vector<E>(A.ncols, E(1.0));
  auto b = mps::spmv(A, xt, KernelMode{});
  SolverConfig cfg;
  cfg.method = KrylovMethod::CG;
  cfg.rel_tol = 1e-20;
  cfg.max_iters = 60;
  // 3. the reference solve_cg over the device operator
  CsrOperator<E> host_op{&A, 16, true};  // thread count does not change bits (test_krylov.cpp:282-300)
  mps::gpu::DeviceCsr<E> dA(A);
  mps::gpu::GpuCsrOperator<E> gop{&dA, 1, true};
  auto ref = mps::solve_cg(host_op, b, cfg);
  auto dev = mps::solve_cg(gop, b, cfg);
  report(ref.report.residual_history == dev.report.residual_history && same_bits(ref.x, dev.x) &&
             ref.report.status == dev.report.status && ref.report.iterations == dev.report.iterations,
         "nd3k K=" + std::to_string(K) + " reference solve_cg over GpuCsrOperator: identical history/x (" +
             std::to_string(ref.report.iterations) + " iterations)");
  // 4. device-resident CG
  auto g = mps::gpu::solve_cg(gop, b, cfg);
  const bool close_iters = std::llabs(g.report.iterations - ref.report.iterations) <= 1;
  report(close_iters && g.report.status == ref.report.status,
         "nd3k K=" + std::to_string(K) + " device solve_cg iterations " + std::to_string(g.report.iterations) +
             " vs reference " + std::to_string(ref.report.iterations));
  const double r = ref.report.final_true_residual, d = g.report.final_true_residual;
  report(d <= 10.0 * r + 1e-30, "nd3k K=" + std::to_string(K) + " device true residual " + sci(d) +
                                   " vs reference " + sci(r));
}

void diag40() {
  using E = MultiComponent<4>;
  CooMatrix<double> coo;
  coo.nrows = coo.ncols = 40;
  for (int i = 0; i < 40; ++i) coo.entries.push_back({i, i, double(i + 1)});
  auto A = convert_csr<E>(coo_to_csr(coo));
  std::vector<E> b(40, E(1.0));
  SolverConfig cfg;
  cfg.rel_tol = 1e-30;
  cfg.max_iters = 200;
  mps::gpu::DeviceCsr<E> dA(A);
  auto g = mps::gpu::solve_cg(mps::gpu::GpuCsrOperator<E>{&dA}, b, cfg);
  report(g.report.converged && g.report.iterations <= 42,  // test_krylov.cpp:94-116: <= k + 2
         "diag(1..40) QD device CG converged in " + std::to_string(g.report.iterations) + " iterations");
}

void errors() {
  auto A = convert_csr<MultiComponent<2>>(example5x5());
  std::vector<MultiComponent<2>> v(4);
  std::string ref_msg, got_msg;
  try {
    mps::spmv(A, v, KernelMode{});
  } catch (const std::invalid_argument& e) {
    ref_msg = e.what();
  }
  try {
    mps::gpu::spmv(A, v, KernelMode{});
  } catch (const std::invalid_argument& e) {
    got_msg = e.what();
  }
  report(!ref_msg.empty() && ref_msg == got_msg, "dimension mismatch message: \"" + got_msg + "\"");
}

template <int K>
void mixed_and_transposed(test::Rng& rng) {
  using E = MultiComponent<K>;
  auto Ad = coo_to_csr(test::random_coo(rng, 600, 600, 15000));  // binary64 matrix
  auto v = random_vector<K>(600, rng);
  for (bool lanes : {true, false}) {
    KernelMode m{{}, MatrixMode::MixedBinary64, false, 3, lanes};
    report(same_bits(mps::spmv(Ad, v, m), mps::gpu::spmv(Ad, v, m)),
           "mixed K=" + std::to_string(K) + (lanes ? " lanes on" : " lanes off") + " spmv bit-exact");
    KernelMode m1{{}, MatrixMode::MixedBinary64, false, 1, lanes};
    report(same_bits(mps::sptmv(Ad, v, m1), mps::gpu::sptmv(Ad, v, m1)),
           "mixed K=" + std::to_string(K) + (lanes ? " lanes on" : " lanes off") + " sptmv bit-exact");
  }
  auto A = full_precision<K>(coo_to_csr(test::random_coo(rng, 500, 700, 12000)), rng);
  auto u = random_vector<K>(500, rng);
  KernelMode one{{}, MatrixMode::Pure, false, 1, true};
  report(same_bits(mps::sptmv(A, u, one), mps::gpu::sptmv(A, u, one)),
         "pure K=" + std::to_string(K) + " sptmv (500x700) bit-exact with the reference at one thread");
  for (int t : {3, 5}) {  // per-thread accumulators merged in thread order (kernels.hpp:368-394)
    KernelMode mt{{}, MatrixMode::Pure, false, t, true};
    report(same_bits(mps::sptmv(A, u, mt), mps::gpu::sptmv(A, u, mt)),
           "pure K=" + std::to_string(K) + " sptmv bit-exact with the reference at " + std::to_string(t) + " threads");
  }
  auto cm = convert_complex_csr<E>(split_complex(test::random_complex_coo(rng, 300, 260, 7000)));
  for (std::size_t i = 0; i < cm.re.indices.size(); ++i) {
    cm.re.values.set(i, rng.multicomp<K>(-4, 4));
    cm.im.values.set(i, rng.multicomp<K>(-4, 4));
  }
  ComplexVector<E> cv{random_vector<K>(300, rng), random_vector<K>(300, rng)};
  for (bool conj : {false, true}) {
    auto r = mps::sptmv_complex(cm, cv, one, conj);
    auto g = mps::gpu::sptmv_complex(cm, cv, one, conj);
    report(same_bits(r.re, g.re) && same_bits(r.im, g.im),
           "complex K=" + std::to_string(K) + (conj ? " adjoint" : " transpose") + " sptmv_complex bit-exact");
    KernelMode m4{{}, MatrixMode::Pure, false, 4, false};
    auto r4 = mps::sptmv_complex(cm, cv, m4, conj);
    auto g4 = mps::gpu::sptmv_complex(cm, cv, m4, conj);
    report(same_bits(r4.re, g4.re) && same_bits(r4.im, g4.im),
           "complex K=" + std::to_string(K) + (conj ? " adjoint" : " transpose") + " sptmv_complex bit-exact at 4 threads");
  }
}

void bicg_over_gpu_operator() {
  using E = MultiComponent<2>;
  test::Rng rng(7);
  auto A = convert_csr<E>(coo_to_csr(test::random_diag_dominant(rng, 300, 0.05, false)));
  auto b = make_vector<E>(A.ncols, E(1.0));
  SolverConfig cfg;
  cfg.method = KrylovMethod::BiCG;
  cfg.rel_tol = 1e-25;
  cfg.max_iters = 200;
  CsrOperator<E> host_op{&A, 1, true};
  mps::gpu::DeviceCsr<E> dA(A, /*with_transpose=*/true);
  mps::gpu::GpuCsrOperator<E> gop{&dA, 1, true};
  auto ref = mps::solve_bicg(host_op, b, cfg);
  auto dev = mps::solve_bicg(gop, b, cfg);
  report(ref.report.residual_history == dev.report.residual_history && same_bits(ref.x, dev.x),
         "reference solve_bicg over GpuCsrOperator (SpMV + SpTMV on the GPU): identical history (" +
             std::to_string(ref.report.iterations) + " iterations)");
}

template <int K>
void device_solvers(test::Rng& rng) {
  using E = MultiComponent<K>;
  for (bool sym : {true, false}) {
    auto Ad = coo_to_csr(test::random_diag_dominant(rng, 400, 0.03, sym));
    auto A = convert_csr<E>(Ad);
    auto b = random_vector<K>(400, rng);
    mps::gpu::DeviceCsr<E> dA(A, /*with_transpose=*/true);
    mps::gpu::DeviceCsr<double, E> dAm(Ad, /*with_transpose=*/true);  // Mixed mode
    for (KrylovMethod m : {KrylovMethod::CG, KrylovMethod::BiCG, KrylovMethod::CGS, KrylovMethod::BiCGSTAB,
                           KrylovMethod::GPBiCG}) {
      if (m == KrylovMethod::CG && !sym) continue;
      for (bool lanes : {true, false}) {
        for (int threads : {1, 4}) {
          if (threads > 1 && m != KrylovMethod::BiCG) continue;
          SolverConfig cfg;
          cfg.method = m;
          cfg.rel_tol = 1e-40;
          cfg.max_iters = 300;
          cfg.lanes_enabled = lanes;
          CsrOperator<E> host_op{&A, threads, lanes};
          mps::gpu::GpuCsrOperator<E> gop{&dA, threads, lanes};
          auto ref = mps::solve(host_op, b, cfg);
          auto dev = mps::gpu::solve(gop, b, cfg, mps::gpu::DotOrder::Sequential);
          const auto& R = ref.report;
          const auto& D = dev.report;
          const std::string tag = std::string(to_string(m)) + " K=" + std::to_string(K) + (sym ? " sym" : " nonsym") +
                                  (lanes ? " lanes on" : " lanes off") + " threads=" + std::to_string(threads);
          report(same_bits(ref.x, dev.x) && R.residual_history == D.residual_history && R.status == D.status &&
                     R.iterations == D.iterations && R.detail == D.detail &&
                     std::bit_cast<std::uint64_t>(R.final_true_residual) ==
                         std::bit_cast<std::uint64_t>(D.final_true_residual),
                 "device solve (sequential dots) bit-exact with mps::solve: " + tag + " (" +
                     std::to_string(R.iterations) + " iterations, " + to_string(R.status) + ")");
          // Mixed mode: CsrOperator<double> over the binary64 matrix (solve_core, bench.cpp:550-557)
          CsrOperator<double> host_opm{&Ad, threads, lanes};
          mps::gpu::GpuCsrOperator<double, E> gopm{&dAm, threads, lanes};
          auto refm = mps::solve(host_opm, b, cfg);
          auto devm = mps::gpu::solve(gopm, b, cfg, mps::gpu::DotOrder::Sequential);
          report(same_bits(refm.x, devm.x) && refm.report.residual_history == devm.report.residual_history &&
                     refm.report.status == devm.report.status && refm.report.detail == devm.report.detail,
                 "device solve (sequential dots) bit-exact with mps::solve, Mixed mode: " + tag + " (" +
                     std::to_string(refm.report.iterations) + " iterations)");
          if (threads == 1 && lanes) {
            auto t = mps::gpu::solve(gop, b, cfg);
            // CG: the north star's +-1%; the Lanczos-type methods amplify round-off
            // (CGS squares the residual polynomial), so +-5% there
            const long long tol = m == KrylovMethod::CG ? std::max<long long>(1, R.iterations / 100)
                                                        : std::max<long long>(2, R.iterations / 20);
            report(t.report.status == R.status && std::llabs(t.report.iterations - R.iterations) <= tol,
                   "device solve (tree dots): " + tag + " " + std::to_string(t.report.iterations) +
                       " iterations vs reference " + std::to_string(R.iterations));
          }
        }
      }
    }
  }
}

}  // namespace

int main() {
  test::Rng rng(20241222);
  spmv_suite<2>(rng);
  spmv_suite<3>(rng);
  spmv_suite<4>(rng);
  complex_suite<2>(rng);
  complex_suite<3>(rng);
  complex_suite<4>(rng);
  solver_suite<2>();
  solver_suite<4>();
  diag40();
  errors();
  mixed_and_transposed<2>(rng);
  mixed_and_transposed<3>(rng);
  mixed_and_transposed<4>(rng);
  bicg_over_gpu_operator();
  device_solvers<2>(rng);
  device_solvers<3>(rng);
  device_solvers<4>(rng);
  std::printf("%d failure(s)\n", failures);
  return failures;
}
