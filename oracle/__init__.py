"""TEST INFRASTRUCTURE ONLY -- the CPU checker, never the product.

ctypes bindings for
  * ``libmpsoracle.so``  the plain-C restatement of the reference path
    (oracle/mpsoracle.c, each function citing the reference file:line), and
  * ``_ref/libmpsref.so`` the UNMODIFIED reference compiled from
    /root/reference by oracle/Makefile (absent on hosts that never had the
    reference; ``ref_available()`` says so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "libmpsoracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libmpsref.so")
REF_V3_SO = os.path.join(_HERE, "_ref", "libmpsref_v3.so")  # same sources, -march=x86-64-v3

_P = ctypes.c_void_p
_i64, _f64, _i32, _u64 = ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_uint64

SCALAR, LANE4 = 0, 1  # lanes off / lanes on (KernelMode::lanes_enabled, kernels.hpp:44)


def _p(a):
    return None if a is None else a.ctypes.data_as(_P)


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------- C restatement
_orc = None


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = ctypes.CDLL(ORACLE_SO)
        for name in ("orc_add", "orc_mul", "orc_sub", "orc_div"):
            getattr(L, name).argtypes = [_i32, _P, _P, _P]
            getattr(L, name).restype = None
        L.orc_mul_d.argtypes = [_i32, _P, _f64, _P]
        L.orc_sqrt.argtypes = [_i32, _P, _P]
        L.orc_to_double.argtypes = [_i32, _P]
        L.orc_to_double.restype = _f64
        L.orc_spmv.argtypes = [_i32, _i32, _i32, _i64, _i64, _i64, _P, _P, _P, _P, _P]
        L.orc_spmv.restype = _i32
        L.orc_spmv_complex.argtypes = [_i32, _i32, _i32, _i64, _i64, _i64, _P, _P, _P, _P, _P, _P, _P, _P]
        L.orc_spmv_complex.restype = _i32
        L.orc_sptmv.argtypes = [_i32, _i32, _i32, _i64, _i64, _i64, _P, _P, _P, _P, _P]
        L.orc_sptmv.restype = _i32
        L.orc_sptmv_complex.argtypes = [_i32, _i32, _i32, _i32, _i64, _i64, _i64, _P, _P, _P, _P, _P, _P, _P,
                                        _P]
        L.orc_sptmv_complex.restype = _i32
        L.orc_checksum.argtypes = [_i32, _i64, _P]
        L.orc_checksum.restype = _u64
        L.orc_checksum_complex.argtypes = [_i32, _i64, _P, _P]
        L.orc_checksum_complex.restype = _u64
        L.orc_exact_diff.argtypes = [_i32, _P, _P]
        L.orc_exact_diff.restype = _f64
        L.orc_exact_diff_vec.argtypes = [_i32, _i64, _P, _P, _P]
        L.orc_exact_diff_vec.restype = None
        L.orc_abs_rowsum.argtypes = [_i32, _i64, _P, _P, _P, _P, _P]
        L.orc_cg.argtypes = [_i32, _i32, _i64, _P, _P, _P, _P, _f64, _f64, _i64, _P, _P, _P, _P,
                             _P, _P]
        L.orc_cg.restype = _i32
        L.orc_solve.argtypes = [_i32, _i32, _i32, _i32, _i64, _P, _P, _P, _P, _P, _f64, _f64, _i64, _P, _P,
                                _P, _P, _P, _P, _P]
        L.orc_solve.restype = _i32
        L.orc_solve_ex.argtypes = [_i32, _i32, _i32, _i32, _i32, _i64, _P, _P, _P, _P, _P, _f64, _f64, _i64, _P,
                                   _P, _P, _P, _P, _P, _P]
        L.orc_solve_ex.restype = _i32
        _orc = L
    return _orc


def mc_op(op: str, K: int, a, b=None):
    a = _c(a)
    out = np.zeros(K)
    L = orc()
    if op == "mul_d":
        L.orc_mul_d(K, _p(a), float(b), _p(out))
    elif op == "sqrt":
        L.orc_sqrt(K, _p(a), _p(out))
    else:
        b = _c(b)
        getattr(L, "orc_" + op)(K, _p(a), _p(b), _p(out))
    return out


def spmv(A, x, order=LANE4, mixed=False):
    """y = A x in the reference order (kernels.hpp:348); A is a synth.HostCsr-like."""
    K = x.shape[1]
    x = _c(x)
    y = np.empty((A.nrows, K))
    vals = _c(A.planes[0] if mixed else A.planes[:K])
    rc = orc().orc_spmv(K, order, 1 if mixed else 0, A.nrows, A.ncols, x.shape[0], _p(_c(A.indptr, np.int64)),
                        _p(_c(A.indices, np.int64)), _p(vals), _p(x), _p(y))
    if rc != 0:
        raise ValueError(f"spmv: vector length {x.shape[0]} does not match matrix dimension {A.ncols}")
    return y


def _cplanes(A, K, mixed):
    """(re, im) value planes of a complex matrix: [K, nnz] each, or one
    binary64 plane each in mixed mode (planes [2, nnz])."""
    P = np.asarray(A.planes)
    return (_c(P[0]), _c(P[1])) if mixed else (_c(P[:K]), _c(P[K:2 * K]))


def spmv_complex(A, xre, xim, order=LANE4, mixed=False):
    K = xre.shape[1]
    yre = np.empty((A.nrows, K))
    yim = np.empty((A.nrows, K))
    vre, vim = _cplanes(A, K, mixed)
    rc = orc().orc_spmv_complex(K, order, 1 if mixed else 0, A.nrows, A.ncols, xre.shape[0],
                                _p(_c(A.indptr, np.int64)), _p(_c(A.indices, np.int64)), _p(vre), _p(vim),
                                _p(_c(xre)), _p(_c(xim)), _p(yre), _p(yim))
    if rc != 0:
        raise ValueError("spmv_complex: dimension mismatch")
    return yre, yim


def sptmv(A, v, threads=1, mixed=False):
    """y = A^T v in the reference's order (kernels.hpp:368-394) for `threads` OpenMP threads."""
    K = v.shape[1]
    y = np.empty((A.ncols, K))
    vals = _c(A.planes[0] if mixed else A.planes[:K])
    rc = orc().orc_sptmv(K, 1 if mixed else 0, threads, A.nrows, A.ncols, v.shape[0], _p(_c(A.indptr, np.int64)),
                         _p(_c(A.indices, np.int64)), _p(vals), _p(_c(v)), _p(y))
    if rc != 0:
        raise ValueError(f"sptmv: vector length {v.shape[0]} does not match matrix dimension {A.nrows}")
    return y


def sptmv_complex(A, vre, vim, threads=1, conjugate=False, mixed=False):
    K = vre.shape[1]
    yre, yim = np.empty((A.ncols, K)), np.empty((A.ncols, K))
    pre, pim = _cplanes(A, K, mixed)
    rc = orc().orc_sptmv_complex(K, 1 if mixed else 0, threads, 1 if conjugate else 0, A.nrows, A.ncols,
                                 vre.shape[0], _p(_c(A.indptr, np.int64)), _p(_c(A.indices, np.int64)), _p(pre),
                                 _p(pim), _p(_c(vre)), _p(_c(vim)), _p(yre), _p(yim))
    if rc != 0:
        raise ValueError("sptmv_complex: dimension mismatch")
    return yre, yim


def checksum(v) -> int:
    v = _c(v)
    K = v.shape[1] if v.ndim == 2 else 1
    return int(orc().orc_checksum(K, v.shape[0], _p(v)))


def checksum_complex(re, im) -> int:
    re, im = _c(re), _c(im)
    return int(orc().orc_checksum_complex(re.shape[1], re.shape[0], _p(re), _p(im)))


def exact_absdiff(a, b) -> np.ndarray:
    """|a_i - b_i| (exact difference, rounded once) for AoS [n,K] arrays."""
    a, b = _c(a), _c(b)
    K = a.shape[1]
    out = np.empty(a.shape[0])
    orc().orc_exact_diff_vec(K, a.shape[0], _p(a), _p(b), _p(out))
    return out


def abs_rowsum(A, lead_plane, x) -> np.ndarray:
    x = _c(x)
    out = np.empty(A.nrows)
    orc().orc_abs_rowsum(x.shape[1], A.nrows, _p(_c(A.indptr, np.int64)), _p(_c(A.indices, np.int64)),
                         _p(_c(lead_plane)), _p(x), _p(out))
    return out


def cg(A, b, order=LANE4, rel_tol=1e-13, abs_tol=1e-99, max_iters=10000):
    K = b.shape[1]
    n = A.nrows
    x = np.zeros((n, K))
    hist = np.zeros(max_iters + 2)
    iters = np.zeros(1, np.int64)
    status = np.zeros(1, np.int32)
    rhs = np.zeros(1)
    tr = np.zeros(1)
    nh = orc().orc_cg(K, order, n, _p(_c(A.indptr, np.int64)), _p(_c(A.indices, np.int64)),
                      _p(_c(A.planes[:K])), _p(_c(b)), rel_tol, abs_tol, max_iters, _p(x), _p(hist),
                      _p(iters), _p(status), _p(rhs), _p(tr))
    return dict(x=x, history=hist[:nh].copy(), iterations=int(iters[0]), status=int(status[0]),
                rhs_norm=float(rhs[0]), final_true_residual=float(tr[0]))


METHODS = ("cg", "bicg", "cgs", "bicgstab", "gpbicg")  # KrylovMethod order, krylov.hpp:24
REASONS = {1: "<p, Ap> vanished", 2: "non-finite residual", 3: "<r~, r> vanished", 4: "<p~, Ap> vanished",
           5: "<r~, Ap> vanished", 6: "<t, t> vanished", 7: "omega vanished", 8: "<At, At> vanished",
           9: "zeta/eta system is singular", 10: "zeta vanished"}


def _method_id(method) -> int:
    return METHODS.index(method) if isinstance(method, str) else int(method)


def detail_text(method, reason: int) -> str:
    return f"{METHODS[_method_id(method)]}: {REASONS[reason]}" if reason else ""


def solve(A, b, method="bicgstab", order=LANE4, threads=1, rel_tol=1e-13, abs_tol=1e-99, max_iters=10000,
          x0=None, mixed=False):
    """C restatement of solve() (krylov.hpp:596-606): every method, sequential
    dots, CsrOperator products (sptmv at `threads`); mixed: A is the binary64
    matrix of CsrOperator<double> (one plane, mul_by_double products)."""
    K = b.shape[1]
    n = A.nrows
    x = np.zeros((n, K))
    hist = np.zeros(max_iters + 2)
    iters = np.zeros(1, np.int64)
    status, reason = np.zeros(1, np.int32), np.zeros(1, np.int32)
    rhs, tr = np.zeros(1), np.zeros(1)
    x0a = None if x0 is None else np.ascontiguousarray(np.asarray(x0, np.float64))
    nh = orc().orc_solve_ex(_method_id(method), K, order, threads, 1 if mixed else 0, n,
                            _p(_c(A.indptr, np.int64)), _p(_c(A.indices, np.int64)),
                            _p(_c(A.planes[:1] if mixed else A.planes[:K])), _p(_c(b)),
                         None if x0a is None else _p(x0a), rel_tol, abs_tol, max_iters, _p(x), _p(hist),
                         _p(iters), _p(status), _p(reason), _p(rhs), _p(tr))
    if nh < 0:
        raise ValueError("solver: invalid configuration")
    return dict(x=x, history=hist[:nh].copy(), iterations=int(iters[0]), status=int(status[0]),
                rhs_norm=float(rhs[0]), final_true_residual=float(tr[0]),
                final_recurrence_residual=float(hist[nh - 1]), detail=detail_text(method, int(reason[0])))


# --------------------------------------------------------------------------- real reference
_ref = None
_ref_path = REF_SO


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def host_has_avx2_fma() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((l for l in f if l.startswith("flags")), "").split()
        return "avx2" in flags and "fma" in flags
    except OSError:
        return False


def use_ref_build(v3: bool) -> bool:
    """Select the reference build later ref() calls use: the reference's own
    flags (default) or the x86-64-v3 build.  Objects made with one build must
    not be passed to the other.  Returns False (and keeps the default) when
    the v3 build or an AVX2+FMA host is missing."""
    global _ref, _ref_path
    want = REF_V3_SO if v3 else REF_SO
    if v3 and not (os.path.exists(REF_V3_SO) and host_has_avx2_fma()):
        return False
    if want != _ref_path:
        _ref, _ref_path = None, want
    return True


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        L = ctypes.CDLL(_ref_path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_csr_create.argtypes = [_i32, _i64, _i64, _P, _P, _P]
        L.ref_csr_create.restype = _P
        L.ref_csr_destroy.argtypes = [_P]
        L.ref_vec_create.argtypes = [_i32, _i64, _P]
        L.ref_vec_create.restype = _P
        L.ref_vec_destroy.argtypes = [_P]
        L.ref_vec_size.argtypes = [_P]
        L.ref_vec_size.restype = _i64
        L.ref_vec_read.argtypes = [_P, _P]
        L.ref_vec_checksum.argtypes = [_P]
        L.ref_vec_checksum.restype = _u64
        L.ref_spmv.argtypes = [_P, _P, _i32, _i32, _P]
        L.ref_spmv.restype = _i32
        L.ref_sptmv.argtypes = [_P, _P, _i32, _i32, _P]
        L.ref_sptmv.restype = _i32
        L.ref_ccsr_create.argtypes = [_i32, _i64, _i64, _P, _P, _P, _P]
        L.ref_ccsr_create.restype = _P
        L.ref_ccsr_destroy.argtypes = [_P]
        L.ref_cvec_create.argtypes = [_i32, _i64, _P, _P]
        L.ref_cvec_create.restype = _P
        L.ref_cvec_destroy.argtypes = [_P]
        L.ref_cvec_read.argtypes = [_P, _P, _P]
        L.ref_cvec_checksum.argtypes = [_P]
        L.ref_cvec_checksum.restype = _u64
        L.ref_spmv_complex.argtypes = [_P, _P, _i32, _i32, _P]
        L.ref_spmv_complex.restype = _i32
        L.ref_sptmv_complex.argtypes = [_P, _P, _i32, _i32, _i32, _P]
        L.ref_sptmv_complex.restype = _i32
        L.ref_mtx_spmv.argtypes = [ctypes.c_char_p, _i32, _i32, _i32, _i32, _i32, _P, _P, _P]
        L.ref_mtx_spmv.restype = _i32
        L.ref_mc_op.argtypes = [_i32, _i32, _P, _P, _P]
        L.ref_make_vector.argtypes = [_i32, _i64, _P]
        L.ref_make_complex_vector.argtypes = [_i32, _i64, _P, _P]
        L.ref_cg.argtypes = [_P, _P, _i32, _i32, _f64, _f64, _i64, _P, _P, _i64, _P, _P, _P, _P, _P,
                             ctypes.c_char_p, _i32]
        L.ref_cg.restype = _i64
        L.ref_solve.argtypes = [_P, _P, _i32, _i32, _i32, _f64, _f64, _i64, _P, _P, _P, _i64, _P, _P, _P,
                                _P, _P, ctypes.c_char_p, _i32]
        L.ref_solve.restype = _i64
        L.ref_fixture.argtypes = [ctypes.c_char_p, _u64, _i64, _i64, _i64]
        L.ref_fixture.restype = _P
        L.ref_csr_info.argtypes = [_P, _P, _P, _P]
        L.ref_csr_export.argtypes = [_P, _P, _P, _P]
        L.ref_csr_export.restype = _i32
        _ref = L
    return _ref


class RefCsr:
    """Reference ``mps::CsrMatrix<E>`` built once (outside any timing)."""

    def __init__(self, A, K, mixed=False):
        self.K = 1 if mixed else K
        vals = _c(A.planes[0] if mixed else A.planes[:K])
        self.h = ref().ref_csr_create(self.K, A.nrows, A.ncols, _p(_c(A.indptr, np.int64)),
                                      _p(_c(A.indices, np.int64)), _p(vals))
        self.nrows = A.nrows

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_csr_destroy(self.h)


class RefVec:
    def __init__(self, x=None, K=None):
        if x is None:
            self.h = ref().ref_vec_create(K, 0, None)
        else:
            x = _c(x)
            self.h = ref().ref_vec_create(x.shape[1], x.shape[0], _p(x))
        self.K = K if x is None else x.shape[1]

    def read(self):
        n = ref().ref_vec_size(self.h)
        out = np.empty((n, self.K))
        ref().ref_vec_read(self.h, _p(out))
        return out

    def checksum(self) -> int:
        return int(ref().ref_vec_checksum(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_vec_destroy(self.h)


def ref_spmv_h(Ah: RefCsr, xh: RefVec, yh: RefVec, order=LANE4, threads=1):
    rc = ref().ref_spmv(Ah.h, xh.h, order, threads, yh.h)
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())


def ref_spmv(A, x, order=LANE4, threads=1, mixed=False):
    K = x.shape[1]
    Ah, xh, yh = RefCsr(A, K, mixed), RefVec(x), RefVec(K=K)
    ref_spmv_h(Ah, xh, yh, order, threads)
    return yh.read()


class RefComplex:
    """Reference ``ComplexSparseMatrix<E>``; mixed: E = double (planes [2, nnz])."""

    def __init__(self, A, K, mixed=False):
        self.K = K
        P = np.asarray(A.planes)
        re_, im_ = (P[0], P[1]) if mixed else (P[:K], P[K:2 * K])
        self.h = ref().ref_ccsr_create(1 if mixed else K, A.nrows, A.ncols, _p(_c(A.indptr, np.int64)),
                                       _p(_c(A.indices, np.int64)), _p(_c(re_)), _p(_c(im_)))

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_ccsr_destroy(self.h)


class RefCVec:
    def __init__(self, re=None, im=None, K=None, n=0):
        if re is None:
            self.h = ref().ref_cvec_create(K, 0, None, None)
            self.K, self.n = K, n
        else:
            re, im = _c(re), _c(im)
            self.h = ref().ref_cvec_create(re.shape[1], re.shape[0], _p(re), _p(im))
            self.K, self.n = re.shape[1], re.shape[0]

    def read(self, n):
        re = np.empty((n, self.K))
        im = np.empty((n, self.K))
        ref().ref_cvec_read(self.h, _p(re), _p(im))
        return re, im

    def checksum(self) -> int:
        return int(ref().ref_cvec_checksum(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_cvec_destroy(self.h)


def ref_mc_op(op: str, K: int, a, b=None):
    code = {"add": 0, "mul": 1, "mul_d": 2, "sub": 3, "div": 4, "sqrt": 5}[op]
    a = _c(a)
    bb = np.zeros(K)
    if op == "mul_d":
        bb[0] = b
    elif b is not None:
        bb = _c(b)
    out = np.zeros(K)
    ref().ref_mc_op(code, K, _p(a), _p(bb), _p(out))
    return out


def ref_make_vector(K, n):
    out = np.empty((n, K))
    ref().ref_make_vector(K, n, _p(out))
    return out


def ref_make_complex_vector(K, n):
    re, im = np.empty((n, K)), np.empty((n, K))
    ref().ref_make_complex_vector(K, n, _p(re), _p(im))
    return re, im


def ref_spmv_complex(A, xr, xi, order=LANE4, threads=1, mixed=False):
    K = xr.shape[1]
    Ah, xh, yh = RefComplex(A, K, mixed), RefCVec(xr, xi), RefCVec(K=K)
    if ref().ref_spmv_complex(Ah.h, xh.h, order, threads, yh.h) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return yh.read(A.nrows)


def ref_sptmv(A, v, order=LANE4, threads=1, mixed=False):
    K = v.shape[1]
    Ah, xh, yh = RefCsr(A, K, mixed), RefVec(v), RefVec(K=K)
    if ref().ref_sptmv(Ah.h, xh.h, order, threads, yh.h) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return yh.read()


def ref_sptmv_complex(A, vr, vi, order=LANE4, threads=1, conjugate=False, mixed=False):
    K = vr.shape[1]
    Ah, xh, yh = RefComplex(A, K, mixed), RefCVec(vr, vi), RefCVec(K=K)
    if ref().ref_sptmv_complex(Ah.h, xh.h, order, threads, 1 if conjugate else 0, yh.h) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return yh.read(A.ncols)


def ref_mtx_spmv(path, K, mixed=False, lanes=True, threads=1, transposed=False):
    """The reference CLI's spmv pipeline on a Matrix Market file (parse_mtx ->
    coo_to_csr / split_complex -> make_vector -> spmv / sptmv -> checksum):
    returns (checksum, n, nnz)."""
    h, n, nz = np.zeros(1, np.uint64), np.zeros(1, np.int64), np.zeros(1, np.int64)
    rc = ref().ref_mtx_spmv(str(path).encode(), K, 1 if mixed else 0, 1 if lanes else 0, threads,
                            1 if transposed else 0, _p(h), _p(n), _p(nz))
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())
    return int(h[0]), int(n[0]), int(nz[0])


def ref_cg(A, b, order=LANE4, threads=1, rel_tol=1e-13, abs_tol=1e-99, max_iters=10000):
    K = b.shape[1]
    Ah, bh = RefCsr(A, K), RefVec(b)
    x = np.zeros((A.nrows, K))
    hist = np.zeros(max_iters + 2)
    iters = np.zeros(1, np.int64)
    status = np.zeros(1, np.int32)
    rhs, tr, fr = np.zeros(1), np.zeros(1), np.zeros(1)
    detail = ctypes.create_string_buffer(256)
    nh = ref().ref_cg(Ah.h, bh.h, order, threads, rel_tol, abs_tol, max_iters, _p(x), _p(hist),
                      len(hist), _p(iters), _p(status), _p(rhs), _p(tr), _p(fr), detail, 256)
    if nh < 0:
        raise ValueError(ref().ref_last_error().decode())
    return dict(x=x, history=hist[:nh].copy(), iterations=int(iters[0]), status=int(status[0]),
                rhs_norm=float(rhs[0]), final_true_residual=float(tr[0]),
                final_recurrence_residual=float(fr[0]), detail=detail.value.decode())


def ref_solve(A, b, method="bicgstab", order=LANE4, threads=1, rel_tol=1e-13, abs_tol=1e-99, max_iters=10000,
              x0=None, mixed=False):
    """The reference solve() itself (oracle/_ref) on the same inputs (mixed:
    CsrOperator<double> over A's leading plane)."""
    K = b.shape[1]
    Ah, bh = RefCsr(A, K, mixed), RefVec(b)
    x = np.zeros((A.nrows, K))
    hist = np.zeros(max_iters + 2)
    iters = np.zeros(1, np.int64)
    status = np.zeros(1, np.int32)
    rhs, tr, fr = np.zeros(1), np.zeros(1), np.zeros(1)
    detail = ctypes.create_string_buffer(256)
    x0a = None if x0 is None else np.ascontiguousarray(np.asarray(x0, np.float64))
    nh = ref().ref_solve(Ah.h, bh.h, _method_id(method), order, threads, rel_tol, abs_tol, max_iters,
                         None if x0a is None else _p(x0a), _p(x), _p(hist), len(hist), _p(iters), _p(status),
                         _p(rhs), _p(tr), _p(fr), detail, 256)
    if nh < 0:
        raise ValueError(ref().ref_last_error().decode())
    return dict(x=x, history=hist[:nh].copy(), iterations=int(iters[0]), status=int(status[0]),
                rhs_norm=float(rhs[0]), final_true_residual=float(tr[0]),
                final_recurrence_residual=float(fr[0]), detail=detail.value.decode())


def ref_fixture(name: str, seed=0, a=0, b=0, c=0):
    """A reference test fixture (tests/support/fixtures.hpp) as int64 CSR + binary64 plane."""
    from types import SimpleNamespace

    h = ref().ref_fixture(name.encode(), seed, a, b, c)
    if not h:
        raise ValueError(name)
    nr, nc, nz = np.zeros(1, np.int64), np.zeros(1, np.int64), np.zeros(1, np.int64)
    ref().ref_csr_info(h, _p(nr), _p(nc), _p(nz))
    indptr = np.empty(int(nr[0]) + 1, np.int64)
    indices = np.empty(int(nz[0]), np.int64)
    vals = np.empty(int(nz[0]))
    ref().ref_csr_export(h, _p(indptr), _p(indices), _p(vals))
    ref().ref_csr_destroy(h)
    return SimpleNamespace(nrows=int(nr[0]), ncols=int(nc[0]), indptr=indptr, indices=indices,
                           planes=vals[None, :], K=1, nnz=int(nz[0]))
