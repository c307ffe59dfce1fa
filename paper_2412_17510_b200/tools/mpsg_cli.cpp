// mpsg_cli.cpp -- the reference CLI's `spmv` and `solve` workflow on the GPU
// (SURVEY 8(f) row 4): Matrix Market in, `mpsparse.bench.v1` /
// `mpsparse.solve.v1` JSON records out, with the same checksum the reference
// prints for the same file, precision, mode and order.
//
//   mpsg spmv  <file.mtx> [--precision dd|td|qd] [--mode p|m] [--lanes on|off|fast]
//              [--threads N] [--reps R] [--transposed] [--matrix-name NAME] [--device D]
//   mpsg solve <file.mtx> [--method cg|bicg|cgs|bicgstab|gpbicg] [--precision ...] [--mode p|m]
//              [--lanes on|off|fast] [--threads N] [--dots tree|exact] [--rtol X] [--atol X]
//              [--max-iters N] [--history FILE] [--matrix-name NAME]
//   (solve: the reference's solve_core, bench.cpp:550-557 -- b = A make_vector,
//   then solve() with the CsrOperator at --threads; --method defaults to
//   bicgstab like the reference CLI, tools/mpsparse.cpp:184.  --dots exact runs
//   the reference's sequential dots: the record then equals the reference's
//   for the same --threads and --lanes, bit for bit.)
//
// Reference workflow restated (paths under /root/reference/proj):
//   parse_mtx            src/mtxio.cpp:85-173 (coordinate real/integer/complex/pattern;
//                        general/symmetric/skew-symmetric/hermitian, expanded as read)
//   coo_to_csr           include/mps/sparse.hpp:80-122 (stable row/col sort, duplicates
//                        summed in input order); split_complex sparse.hpp:240-252
//   convert_csr          sparse.hpp:195-207 (exact widening to K components)
//   make_vector          bench.hpp:78-111 -> mpsg_make_vector (device, reference bits)
//   time_real_loop       src/bench.cpp:54-85 (one warm-up, median of R timed calls)
//   BenchRecord::to_json src/bench.cpp:139-152; solve record src/bench.cpp:602-619
//   run_spmv / run_solve tools/mpsparse.cpp:74-134
// The matrix is uploaded once (outside the timing, as the reference converts
// before timing, bench.cpp:211-213); each timed call is the host-pointer SpMV.
// --threads is recorded; it changes nothing for spmv (rows are independent)
// and selects the reference's thread-order merge for sptmv (kernels.hpp:368-394),
// reproduced bit for bit.  --lanes fast selects the throughput order.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <thread>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mpsg.h"

namespace {

struct Coo {
  int64_t nrows = 0, ncols = 0;
  bool complex = false;
  std::vector<int64_t> r, c;
  std::vector<double> re, im;
};

[[noreturn]] void die(const std::string& msg, int code = 2) {
  std::fprintf(stderr, "mpsg: %s\n", msg.c_str());
  std::exit(code);
}

bool content_line(std::istream& in, std::string& line, size_t& lineno) {
  while (std::getline(in, line)) {
    ++lineno;
    size_t i = line.find_first_not_of(" \t\r\n\v\f");
    if (i == std::string::npos || line[i] == '%') continue;
    return true;
  }
  return false;
}

// src/mtxio.cpp:85-173
Coo parse_mtx(const std::string& path) {
  std::ifstream in(path);
  if (!in) die("cannot open " + path);
  std::string line;
  size_t lineno = 0;
  if (!std::getline(in, line)) die("matrix market, line 1: empty stream");
  ++lineno;
  std::string lo = line;
  std::transform(lo.begin(), lo.end(), lo.begin(), [](unsigned char ch) { return (char)std::tolower(ch); });
  std::istringstream hdr(lo);
  std::string banner, object, format, field, sym;
  hdr >> banner >> object >> format >> field >> sym;
  if (banner != "%%matrixmarket" || object != "matrix") die("matrix market, line 1: missing %%MatrixMarket banner");
  if (format != "coordinate") die("matrix market, line 1: only coordinate format is supported");
  if (field != "real" && field != "integer" && field != "complex" && field != "pattern")
    die("matrix market, line 1: unknown field '" + field + "'");
  if (sym != "general" && sym != "symmetric" && sym != "skew-symmetric" && sym != "hermitian")
    die("matrix market, line 1: unknown symmetry '" + sym + "'");
  if (sym == "hermitian" && field != "complex") die("matrix market, line 1: hermitian requires a complex field");
  if (!content_line(in, line, lineno)) die("matrix market: missing size line");
  Coo m;
  long long nr = 0, nc = 0, nz = 0;
  {
    std::istringstream ss(line);
    if (!(ss >> nr >> nc >> nz)) die("matrix market, line " + std::to_string(lineno) + ": bad size line");
  }
  if (nr <= 0 || nc <= 0 || nz < 0) die("matrix market: invalid dimensions");
  if (nr != nc) die("matrix is " + std::to_string(nr) + "x" + std::to_string(nc) + " but a square matrix is required");
  m.nrows = nr;
  m.ncols = nc;
  m.complex = field == "complex";
  const bool general = sym == "general";
  for (long long seen = 0; seen < nz; ++seen) {
    if (!content_line(in, line, lineno))
      die("matrix market: expected " + std::to_string(nz) + " entries, found " + std::to_string(seen));
    const char* p = line.c_str();
    // parse_index / parse_value / expect_line_end (mtxio.cpp:40-66): a number
    // must be present and in range, nothing may follow the entry
    auto bad = [&](const char* what) { die("matrix market, line " + std::to_string(lineno) + ": " + what); };
    auto index = [&]() -> long long {
      errno = 0;
      char* end = nullptr;
      const long long v = std::strtoll(p, &end, 10);
      if (end == p || errno == ERANGE) bad("expected integer");
      p = end;
      return v;
    };
    auto value = [&]() -> double {
      errno = 0;
      char* end = nullptr;
      const double v = std::strtod(p, &end);
      if (end == p || errno == ERANGE) bad("expected number");
      p = end;
      return v;
    };
    const long long r = index() - 1;
    const long long c = index() - 1;
    if (r < 0 || r >= nr || c < 0 || c >= nc) die("matrix market, line " + std::to_string(lineno) + ": index out of range");
    double re = 1.0, im = 0.0;
    if (field != "pattern") re = value();
    if (m.complex) {
      im = value();
      if (sym == "hermitian" && r == c && im != 0.0) die("matrix market: hermitian diagonal must be real");
    }
    for (; *p; ++p)
      if (!std::isspace(static_cast<unsigned char>(*p))) bad("trailing characters after entry");
    if (!general && c > r) die("matrix market: entry above the diagonal in a symmetric-format matrix");
    // append_expanded (mtxio.cpp:67-81): the entry, then its mirror
    m.r.push_back(r), m.c.push_back(c), m.re.push_back(re), m.im.push_back(im);
    if (!general && r != c) {
      double mre = re, mim = sym == "hermitian" ? -im : im;
      if (sym == "skew-symmetric") mre = -mre, mim = -mim;
      m.r.push_back(c), m.c.push_back(r), m.re.push_back(mre), m.im.push_back(mim);
    }
  }
  if (content_line(in, line, lineno)) die("matrix market: more entries than declared");
  return m;
}

struct Csr {
  int64_t nrows = 0, ncols = 0;
  std::vector<int64_t> indptr, indices;
  std::vector<double> re, im;  // binary64 values (re / im parts)
};

// sparse.hpp:80-122 (applied to the re and im parts alike: split_complex
// builds two COO matrices over the same entry list)
Csr coo_to_csr(const Coo& m) {
  std::vector<size_t> order(m.r.size());
  std::iota(order.begin(), order.end(), size_t{0});
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return m.r[a] != m.r[b] ? m.r[a] < m.r[b] : m.c[a] < m.c[b];
  });
  Csr a;
  a.nrows = m.nrows;
  a.ncols = m.ncols;
  a.indptr.assign((size_t)m.nrows + 1, 0);
  int64_t pr = -1, pc = -1;
  for (size_t oi : order) {
    if (m.r[oi] == pr && m.c[oi] == pc) {
      a.re.back() = a.re.back() + m.re[oi];
      a.im.back() = a.im.back() + m.im[oi];
      continue;
    }
    a.re.push_back(m.re[oi]);
    a.im.push_back(m.im[oi]);
    a.indices.push_back(m.c[oi]);
    a.indptr[(size_t)m.r[oi] + 1]++;
    pr = m.r[oi];
    pc = m.c[oi];
  }
  for (size_t i = 1; i < a.indptr.size(); ++i) a.indptr[i] += a.indptr[i - 1];
  return a;
}

void check(mpsg_ctx* ctx, int rc, const char* what) {
  if (rc != MPSG_OK) die(std::string(what) + ": " + mpsg_last_error(ctx), 1);
}

double median(std::vector<double> v) {  // bench.cpp median_of
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o + "\"";
}
std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

struct Args {
  std::string cmd, path, precision = "dd", mode = "p", lanes = "on", name, method = "bicgstab", history,
      dots = "tree";
  int threads = 0, reps = 5, device = 0;
  bool transposed = false;
  double rtol = 1e-13, atol = 1e-99;
  int64_t max_iters = 10000;
};

Args parse_args(int argc, char** argv) {
  if (argc < 3) die("usage: mpsg spmv|solve <file.mtx> [options]  (see the file header)");
  Args a;
  a.cmd = argv[1];
  a.path = argv[2];
  for (int i = 3; i < argc; ++i) {
    std::string o = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) die("missing value for " + o);
      return argv[++i];
    };
    if (o == "--precision") a.precision = val();
    else if (o == "--mode") a.mode = val();
    else if (o == "--lanes") a.lanes = val();
    else if (o == "--threads") a.threads = std::atoi(val().c_str());
    else if (o == "--reps") a.reps = std::atoi(val().c_str());
    else if (o == "--transposed") a.transposed = true;
    else if (o == "--matrix-name") a.name = val();
    else if (o == "--device") a.device = std::atoi(val().c_str());
    else if (o == "--method") a.method = val();
    else if (o == "--rtol") a.rtol = std::atof(val().c_str());
    else if (o == "--atol") a.atol = std::atof(val().c_str());
    else if (o == "--max-iters") a.max_iters = std::atoll(val().c_str());
    else if (o == "--history") a.history = val();
    else if (o == "--dots") a.dots = val();
    else die("unknown option " + o);
  }
  if (a.name.empty()) {
    size_t s = a.path.find_last_of('/');
    std::string base = s == std::string::npos ? a.path : a.path.substr(s + 1);
    size_t d = base.find_last_of('.');
    a.name = d == std::string::npos ? base : base.substr(0, d);
  }
  return a;
}

int precision_k(const std::string& p) {
  if (p == "dd") return 2;
  if (p == "td") return 3;
  if (p == "qd") return 4;
  die("precision '" + p + "': the device runs dd, td and qd");
}

int order_of(const std::string& lanes) {
  if (lanes == "on") return MPSG_ORDER_LANE4;
  if (lanes == "off") return MPSG_ORDER_SCALAR;
  if (lanes == "fast") return MPSG_ORDER_FAST;
  die("--lanes must be on, off or fast");
}

mpsg_csr* upload(mpsg_ctx* ctx, const Csr& A, int K, bool cplx, bool mixed, bool transpose) {
  const int per = mixed ? 1 : K;
  std::vector<std::vector<double>> planes;
  const int64_t nnz = (int64_t)A.indices.size();
  for (int part = 0; part < (cplx ? 2 : 1); ++part) {
    const std::vector<double>& v = part == 0 ? A.re : A.im;
    planes.push_back(v);  // leading component: the binary64 value
    for (int j = 1; j < per; ++j) planes.push_back(std::vector<double>((size_t)nnz, 0.0));  // convert_csr: exact
  }
  std::vector<const double*> pp;
  for (auto& p : planes) pp.push_back(p.data());
  const int flags = (cplx ? MPSG_CSR_COMPLEX : 0) | (mixed ? MPSG_CSR_MIXED : 0) | (transpose ? MPSG_CSR_TRANSPOSE : 0);
  mpsg_csr* d = nullptr;
  check(ctx, mpsg_csr_upload_ex(ctx, K, flags, A.nrows, A.ncols, A.indptr.data(), A.indices.data(), pp.data(), &d),
        "upload");
  return d;
}

// Context creation, retried a few times: a device-initialisation failure can be
// transient while another process on the GPU is tearing its context down.
// mpsg_ctx_create owns the retry policy (a device briefly held by another
// process); anything it cannot recover from is reported with the CUDA text.
static mpsg_ctx* open_ctx(int device) {
  mpsg_ctx* ctx = nullptr;
  if (mpsg_ctx_create(device, &ctx) != MPSG_OK) die(std::string("no usable sm_100a GPU: ") + mpsg_create_error(), 1);
  return ctx;
}

int run_spmv(const Args& a) {
  const Coo coo = parse_mtx(a.path);
  const Csr A = coo_to_csr(coo);
  const int K = precision_k(a.precision);
  if (a.mode != "p" && a.mode != "m") die("--mode must be p or m");
  const bool mixed = a.mode == "m", cplx = coo.complex;
  const int order = order_of(a.lanes);
  if (a.reps < 1) die("time_kernel: repetitions must be at least 1");
  mpsg_ctx* ctx = open_ctx(a.device);
  mpsg_csr* d = upload(ctx, A, K, cplx, mixed, a.transposed);
  const int64_t n = A.ncols;
  std::vector<double> vr((size_t)n * K), vi(cplx ? (size_t)n * K : 0), yr((size_t)n * K), yi(vi.size());
  check(ctx, mpsg_make_vector(ctx, K, n, vr.data(), cplx ? vi.data() : nullptr), "make_vector");
  auto run = [&] {
    int rc;
    const int thr = a.threads > 0 ? a.threads : 1;  // sptmv's bits depend on the thread count
    if (cplx)
      rc = a.transposed
               ? mpsg_sptmv_complex_ex(ctx, d, order, thr, 0, n, vr.data(), vi.data(), yr.data(), yi.data())
               : mpsg_spmv_complex(ctx, d, order, n, vr.data(), vi.data(), yr.data(), yi.data());
    else
      rc = a.transposed ? mpsg_sptmv_ex(ctx, d, order, thr, n, vr.data(), yr.data())
                        : mpsg_spmv(ctx, d, order, n, vr.data(), yr.data());
    check(ctx, rc, "spmv");
  };
  run();  // warm-up (bench.cpp:59)
  std::vector<double> times;
  for (int i = 0; i < a.reps; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    run();
    times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  const uint64_t h = cplx ? mpsg_checksum_complex(K, n, yr.data(), yi.data()) : mpsg_checksum(K, n, yr.data());
  const char* kernel = cplx ? (a.transposed ? "sptmv_complex" : "spmv_complex") : (a.transposed ? "sptmv" : "spmv");
  char hex[20];
  std::snprintf(hex, sizeof(hex), "%016" PRIx64, h);
  std::printf("{\"schema\":\"mpsparse.bench.v1\",\"matrix\":%s,\"n\":%lld,\"nnz\":%lld,\"kernel\":\"%s\","
              "\"precision\":\"%s\",\"mode\":\"%s\",\"threads\":%d,\"lanes\":%s,\"repetitions\":%d,"
              "\"median_seconds\":%s,\"checksum\":\"%s\",\"device\":\"%s\",\"order\":\"%s\"}\n",
              jstr(a.name).c_str(), (long long)A.nrows, (long long)A.indices.size(), kernel, a.precision.c_str(),
              a.mode.c_str(), a.threads > 0 ? a.threads : 1, a.lanes == "off" ? "false" : "true", a.reps,
              jnum(median(times)).c_str(), hex, mpsg_version(), a.lanes.c_str());
  mpsg_csr_destroy(d);
  mpsg_ctx_destroy(ctx);
  return 0;
}

int run_solve(const Args& a) {
  static const char* methods[] = {"cg", "bicg", "cgs", "bicgstab", "gpbicg"};  // parse_method, krylov.hpp:37-44
  int method = -1;
  for (int m = 0; m < 5; ++m)
    if (a.method == methods[m]) method = m;
  if (method < 0) die("solve: unknown method '" + a.method + "' (cg, bicg, cgs, bicgstab, gpbicg)");
  if (a.dots != "tree" && a.dots != "exact") die("solve: --dots is tree or exact");
  const Coo coo = parse_mtx(a.path);
  if (coo.complex) die("solve: complex matrices are not supported; the solvers are real", 1);
  if (a.mode != "p" && a.mode != "m") die("solve: --mode is p (Pure) or m (Mixed)");
  const bool mixed = a.mode == "m";
  const Csr A = coo_to_csr(coo);
  if (A.nrows != A.ncols) die("solve: the matrix must be square", 1);
  const int K = precision_k(a.precision);
  mpsg_ctx* ctx = open_ctx(a.device);
  mpsg_csr* d = upload(ctx, A, K, false, mixed, method == MPSG_BICG);
  const int64_t n = A.ncols;
  const int threads = a.threads > 0 ? a.threads : 1;
  std::vector<double> v((size_t)n * K), b((size_t)n * K), x((size_t)n * K), hist((size_t)a.max_iters + 1);
  check(ctx, mpsg_make_vector(ctx, K, n, v.data(), nullptr), "make_vector");
  const int order = order_of(a.lanes);
  check(ctx, mpsg_spmv(ctx, d, order, n, v.data(), b.data()), "spmv");  // b = A v (bench.cpp:552-554)
  mpsg_cg_report rep{};
  if (method == MPSG_CG && a.dots == "tree") {
    mpsg_cg_config cfg{a.rtol, a.atol, a.max_iters, 32, 1};
    check(ctx, mpsg_cg(ctx, d, order, n, b.data(), nullptr, &cfg, x.data(), hist.data(), (int64_t)hist.size(), &rep),
          "cg");
  } else {
    mpsg_solver_config cfg{};
    cfg.method = method;
    cfg.threads = threads;
    cfg.rel_tol = a.rtol;
    cfg.abs_tol = a.atol;
    cfg.max_iters = a.max_iters;
    cfg.check_every = 32;
    cfg.use_graph = 1;
    cfg.dot_order = a.dots == "exact" ? MPSG_DOT_SEQUENTIAL : MPSG_DOT_TREE;
    check(ctx, mpsg_solve(ctx, d, order, n, b.data(), nullptr, &cfg, x.data(), hist.data(), (int64_t)hist.size(),
                          &rep),
          "solve");
  }
  static const char* status[] = {"converged", "max_iterations", "breakdown", "diverged"};
  if (!a.history.empty()) {
    std::ofstream h(a.history);
    h << "iter,residual\n";
    for (int64_t k = 0; k < rep.history_len; ++k) h << k << ',' << jnum(hist[(size_t)k]) << '\n';
  }
  std::printf("{\"schema\":\"mpsparse.solve.v1\",\"matrix\":%s,\"method\":\"%s\",\"precision\":\"%s\","
              "\"mode\":\"%s\",\"threads\":%d,\"n\":%lld,\"nnz\":%lld,\"status\":\"%s\",\"converged\":%s,"
              "\"iterations\":%lld,\"rhs_norm\":%s,\"final_recurrence_residual\":%s,\"final_true_residual\":%s,"
              "\"setup_seconds\":%s,\"solve_seconds\":%s%s%s%s}\n",
              jstr(a.name).c_str(), methods[method], a.precision.c_str(), mixed ? "m" : "p", threads, (long long)A.nrows,
              (long long)A.indices.size(), status[rep.status], rep.converged ? "true" : "false",
              (long long)rep.iterations, jnum(rep.rhs_norm).c_str(), jnum(rep.final_recurrence_residual).c_str(),
              jnum(rep.final_true_residual).c_str(), jnum(rep.setup_seconds).c_str(),
              jnum(rep.solve_seconds).c_str(), rep.detail[0] ? ",\"detail\":" : "",
              rep.detail[0] ? jstr(rep.detail).c_str() : "",
              a.history.empty() ? "" : (",\"residual_csv\":" + jstr(a.history)).c_str());
  mpsg_csr_destroy(d);
  mpsg_ctx_destroy(ctx);
  return rep.converged ? 0 : 3;
}

}  // namespace

int main(int argc, char** argv) {
  const Args a = parse_args(argc, argv);
  if (a.cmd == "spmv") return run_spmv(a);
  if (a.cmd == "solve") return run_solve(a);
  die("unknown subcommand '" + a.cmd + "' (spmv, solve)");
}
