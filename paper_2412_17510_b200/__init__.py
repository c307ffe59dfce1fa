"""B200-native multi-precision CSR SpMV (DD/TD/QD, real and complex) and CG.

Host-side mirror of the reference's interface for this path, calling the
CUDA library ``libmpsg.so`` through its C ABI (include/mpsg.h).  Names,
argument meaning and error behaviour follow the reference
(/root/reference/proj/include/mps/):

  reference                                   here
  ------------------------------------------  ------------------------------------
  CsrMatrix<E> (sparse.hpp:69-78)              DeviceCsr (uploaded once)
  KernelMode (kernels.hpp:39-45)               KernelMode (threads ignored; lanes
                                               selects LANE4 / SCALAR; fast=True
                                               selects the throughput order)
  spmv(A, v, mode) (kernels.hpp:348)           spmv(A, v, mode)
  spmv_complex(A, v, mode) (kernels.hpp:399)   spmv_complex(A, v_re, v_im, mode)
  CsrOperator (krylov.hpp:101-120)             CsrOperator
  SolverConfig / SolverReport (krylov.hpp)     SolverConfig / SolverReport
  solve_cg(op, b, cfg) (krylov.hpp:238)        solve_cg(op, b, cfg)
  solve(op, b, cfg) (krylov.hpp:596-606)       solve(op, b, cfg) -- cfg.method picks
  solve_bicg/cgs/bicgstab/gpbicg (:283-594)    solve_bicg / solve_cgs / solve_bicgstab /
                                               solve_gpbicg (device-resident)
  KrylovMethod / parse_method (krylov.hpp:24)  KrylovMethod / parse_method
  partition_rows (kernels.hpp:63-80)           partition_rows
  checksum (bench.hpp:113-150)                 checksum / checksum_complex

Vectors are numpy float64 arrays of shape (n, K): the memory image of
``std::vector<MultiComponent<K>>``.  ``std::invalid_argument`` becomes
``ValueError`` with the reference's message text.  There is no CPU
fallback: if the CUDA library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import enum
import os
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPSG_LIB") or os.path.join(_HERE, "libmpsg.so")

ORDER_SCALAR, ORDER_LANE4, ORDER_FAST = 0, 1, 2
E_OK, E_DIM, E_RANGE, E_CUDA, E_NCCL, E_OOM, E_ARG, E_STRUCT = range(8)

_P = ctypes.c_void_p
_i64, _i32, _f64, _u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64


class MpsgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[mpsg error {code}] {msg}")
        self.code = code


class CsrStats(ctypes.Structure):
    _fields_ = [("nrows", _i64), ("ncols", _i64), ("nnz", _i64), ("K", ctypes.c_int32),
                ("is_complex", ctypes.c_int32), ("nslices", _i64), ("sell_elems", _i64),
                ("nlong", _i64), ("long_nnz", _i64), ("nchunks", _i64), ("device_bytes", _i64),
                ("is_mixed", ctypes.c_int32), ("has_transpose", ctypes.c_int32)]


class _CgConfig(ctypes.Structure):
    _fields_ = [("rel_tol", _f64), ("abs_tol", _f64), ("max_iters", _i64),
                ("check_every", ctypes.c_int32), ("use_graph", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class _SolverConfig(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("threads", ctypes.c_int32), ("rel_tol", _f64), ("abs_tol", _f64),
                ("max_iters", _i64), ("check_every", ctypes.c_int32), ("use_graph", ctypes.c_int32),
                ("dot_order", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class _CgReport(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("converged", ctypes.c_int32), ("iterations", _i64),
                ("history_len", _i64), ("rhs_norm", _f64), ("final_recurrence_residual", _f64),
                ("final_true_residual", _f64), ("setup_seconds", _f64), ("solve_seconds", _f64),
                ("detail", ctypes.c_char * 64), ("device_seconds", _f64)]


_lib = None

# every symbol include/mpsg.h declares
EXPORTS = ("mpsg_ctx_create", "mpsg_create_error", "mpsg_ctx_destroy", "mpsg_last_error", "mpsg_ctx_set_stream",
           "mpsg_ctx_set_layout", "mpsg_ctx_synchronize", "mpsg_csr_upload", "mpsg_csr_destroy",
           "mpsg_csr_get_stats", "mpsg_spmv", "mpsg_spmv_dev", "mpsg_spmv_complex",
           "mpsg_spmv_complex_dev", "mpsg_cg", "mpsg_partition_rows", "mpsg_checksum",
           "mpsg_checksum_complex", "mpsg_version", "mpsg_measure_fp64_peak", "mpsg_mc_op_dev",
           "mpsg_comm_unique_id", "mpsg_comm_create", "mpsg_comm_destroy", "mpsg_dcsr_upload",
           "mpsg_dcsr_destroy", "mpsg_dcsr_info", "mpsg_dspmv", "mpsg_dspmv_dev", "mpsg_dspmv_complex_dev",
           "mpsg_dcg", "mpsg_halo_plan", "mpsg_csr_upload_ex", "mpsg_sptmv", "mpsg_sptmv_dev",
           "mpsg_sptmv_complex", "mpsg_sptmv_complex_dev", "mpsg_comm_create_local", "mpsg_make_vector",
           "mpsg_sptmv_ex", "mpsg_sptmv_complex_ex", "mpsg_solve", "mpsg_dsolve", "mpsg_dcsr_interior_rows")

CSR_COMPLEX, CSR_MIXED, CSR_TRANSPOSE = 1, 2, 4


def lib():
    """Load libmpsg.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          "(make -C paper_2412_17510_b200/csrc)")
    L = ctypes.CDLL(LIB_PATH)
    L.mpsg_ctx_create.argtypes = [_i32, ctypes.POINTER(_P)]
    L.mpsg_ctx_destroy.argtypes = [_P]
    L.mpsg_create_error.argtypes = []
    L.mpsg_create_error.restype = ctypes.c_char_p
    L.mpsg_last_error.argtypes = [_P]
    L.mpsg_last_error.restype = ctypes.c_char_p
    L.mpsg_ctx_set_stream.argtypes = [_P, _P]
    L.mpsg_ctx_set_layout.argtypes = [_P, _i64, _i64, _i64]
    L.mpsg_ctx_synchronize.argtypes = [_P]
    L.mpsg_csr_upload.argtypes = [_P, _i32, _i32, _i64, _i64, _P, _P, ctypes.POINTER(_P),
                                  ctypes.POINTER(_P)]
    L.mpsg_csr_destroy.argtypes = [_P]
    L.mpsg_csr_get_stats.argtypes = [_P, ctypes.POINTER(CsrStats)]
    L.mpsg_spmv.argtypes = [_P, _P, _i32, _i64, _P, _P]
    L.mpsg_spmv_dev.argtypes = [_P, _P, _i32, _P, _P, _P]
    L.mpsg_spmv_complex.argtypes = [_P, _P, _i32, _i64, _P, _P, _P, _P]
    L.mpsg_spmv_complex_dev.argtypes = [_P, _P, _i32, _P, _P, _P, _P, _P]
    L.mpsg_cg.argtypes = [_P, _P, _i32, _i64, _P, _P, ctypes.POINTER(_CgConfig), _P, _P, _i64,
                          ctypes.POINTER(_CgReport)]
    L.mpsg_solve.argtypes = [_P, _P, _i32, _i64, _P, _P, ctypes.POINTER(_SolverConfig), _P, _P, _i64,
                             ctypes.POINTER(_CgReport)]
    L.mpsg_dcsr_interior_rows.argtypes = [_P, _P]
    L.mpsg_dsolve.argtypes = [_P, _i32, _P, _P, ctypes.POINTER(_SolverConfig), _P, _P, _i64,
                              ctypes.POINTER(_CgReport)]
    L.mpsg_partition_rows.argtypes = [_P, _i64, _i32, _P]
    L.mpsg_checksum.argtypes = [_i32, _i64, _P]
    L.mpsg_checksum.restype = _u64
    L.mpsg_checksum_complex.argtypes = [_i32, _i64, _P, _P]
    L.mpsg_checksum_complex.restype = _u64
    L.mpsg_version.restype = ctypes.c_char_p
    L.mpsg_measure_fp64_peak.argtypes = [_P, ctypes.POINTER(_f64)]
    L.mpsg_mc_op_dev.argtypes = [_P, _i32, _i32, _i64, _P, _P, _P]
    L.mpsg_comm_unique_id.argtypes = [_P]
    L.mpsg_comm_create.argtypes = [_P, _i32, _i32, _P, ctypes.POINTER(_P)]
    L.mpsg_comm_destroy.argtypes = [_P]
    L.mpsg_comm_create_local.argtypes = [ctypes.POINTER(_P), _i32, ctypes.POINTER(_P)]
    L.mpsg_make_vector.argtypes = [_P, _i32, _i64, _P, _P]
    L.mpsg_sptmv_ex.argtypes = [_P, _P, _i32, _i32, _i64, _P, _P]
    L.mpsg_sptmv_complex_ex.argtypes = [_P, _P, _i32, _i32, _i32, _i64, _P, _P, _P, _P]
    L.mpsg_dcsr_upload.argtypes = [_P, _i32, _i32, _i64, _i64, _i64, _P, _P, ctypes.POINTER(_P),
                                   ctypes.POINTER(_P)]
    L.mpsg_dcsr_destroy.argtypes = [_P]
    L.mpsg_dcsr_info.argtypes = [_P, _P, _P]
    L.mpsg_dspmv.argtypes = [_P, _i32, _P, _P]
    L.mpsg_dspmv_dev.argtypes = [_P, _i32, _P, _P, _P]
    L.mpsg_dspmv_complex_dev.argtypes = [_P, _i32, _P, _P, _P, _P, _P]
    L.mpsg_dcg.argtypes = [_P, _i32, _P, _P, ctypes.POINTER(_CgConfig), _P, _P, _i64,
                           ctypes.POINTER(_CgReport)]
    L.mpsg_halo_plan.argtypes = [_i32, _i32, _P, _P, _P, _P]
    L.mpsg_csr_upload_ex.argtypes = [_P, _i32, _i32, _i64, _i64, _P, _P, ctypes.POINTER(_P), ctypes.POINTER(_P)]
    L.mpsg_sptmv.argtypes = [_P, _P, _i32, _i64, _P, _P]
    L.mpsg_sptmv_dev.argtypes = [_P, _P, _i32, _P, _P, _P]
    L.mpsg_sptmv_complex.argtypes = [_P, _P, _i32, _i32, _i64, _P, _P, _P, _P]
    L.mpsg_sptmv_complex_dev.argtypes = [_P, _P, _i32, _i32, _P, _P, _P, _P, _P]
    _lib = L
    return L


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_P)


def _aos(v, name="vector", K: int | None = None) -> np.ndarray:
    """(n, K) float64 C-contiguous view of v.  With K given, the component
    count must match the matrix: the C ABI copies n*K doubles each way, so a
    narrower vector would be read (and its result written) past its end."""
    a = np.ascontiguousarray(v, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] not in (2, 3, 4):
        raise ValueError(f"{name}: expected an (n, K) float64 array with K in 2..4, got {a.shape}")
    if K is not None and a.shape[1] != K:
        raise ValueError(f"{name}: vector has K={a.shape[1]} components, matrix has K={K}")
    return a


# --------------------------------------------------------------------------- context
class Context:
    """One device, one stream (mpsg_ctx).  Not thread-safe, like the C ABI."""

    def __init__(self, device: int = 0):
        self.device = device
        h = _P()
        rc = lib().mpsg_ctx_create(device, ctypes.byref(h))
        if rc != E_OK:
            raise MpsgError(rc, f"no usable sm_100a GPU: {lib().mpsg_create_error().decode()}")
        self.h = h

    def check(self, rc: int):
        if rc == E_OK:
            return
        msg = lib().mpsg_last_error(self.h).decode()
        if rc == E_DIM:
            raise ValueError(msg)
        raise MpsgError(rc, msg)

    def set_stream(self, stream_ptr: int | None):
        self.check(lib().mpsg_ctx_set_stream(self.h, stream_ptr))

    def set_layout(self, long_threshold=0, sigma=0, fast_chunk=0):
        self.check(lib().mpsg_ctx_set_layout(self.h, long_threshold, sigma, fast_chunk))

    def synchronize(self):
        self.check(lib().mpsg_ctx_synchronize(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().mpsg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("MPSG_DEVICE", "0")))
    return _default_ctx


# --------------------------------------------------------------------------- matrices
class DeviceCsr:
    """Device copy of a reference CSR (``CsrMatrix<MultiComponent<K>>`` or a
    ``ComplexSparseMatrix`` sharing one structure).

    ``A`` is any object with ``nrows, ncols, indptr (int64), indices (int64),
    planes``: [K, nnz] real, [2K, nnz] complex (re planes then im planes);
    with ``mixed`` (the binary64 matrix of Mixed mode, ``CsrMatrix<double>``)
    one plane real, two complex.  ``transpose`` also uploads A^T for sptmv.
    """

    def __init__(self, A, K: int, is_complex: bool = False, ctx: Optional[Context] = None,
                 mixed: bool = False, transpose: bool = False):
        self.ctx = ctx or default_context()
        self.K = K
        self.is_complex = bool(is_complex)
        self.mixed = bool(mixed)
        self.nrows, self.ncols = int(A.nrows), int(A.ncols)
        indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(A.indices, dtype=np.int64)
        nplanes = (1 if mixed else K) * (2 if is_complex else 1)
        planes = np.asarray(A.planes)
        if planes.shape[0] < nplanes:
            raise ValueError(f"DeviceCsr: need {nplanes} value planes, got {planes.shape[0]}")
        plist = [np.ascontiguousarray(planes[j], dtype=np.float64) for j in range(nplanes)]
        parr = (_P * nplanes)(*[p.ctypes.data for p in plist])
        flags = (CSR_COMPLEX if is_complex else 0) | (CSR_MIXED if mixed else 0) | (CSR_TRANSPOSE if transpose else 0)
        h = _P()
        self.ctx.check(lib().mpsg_csr_upload_ex(self.ctx.h, K, flags, self.nrows, self.ncols, _p(indptr),
                                                _p(indices), parr, ctypes.byref(h)))
        self.h = h
        self.nnz = int(indptr[-1])

    def stats(self) -> CsrStats:
        s = CsrStats()
        self.ctx.check(lib().mpsg_csr_get_stats(self.h, ctypes.byref(s)))
        return s

    def close(self):
        if getattr(self, "h", None):
            lib().mpsg_csr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class KernelMode:
    """kernels.hpp:39-45.  ``threads`` has no device meaning; ``lanes_enabled``
    picks the bit-exact order; ``fast`` picks the throughput order."""

    threads: int = 1
    lanes_enabled: bool = True
    fast: bool = False

    @property
    def order(self) -> int:
        if self.fast:
            return ORDER_FAST
        return ORDER_LANE4 if self.lanes_enabled else ORDER_SCALAR


def _order(mode) -> int:
    if mode is None:
        return ORDER_LANE4
    if isinstance(mode, int):
        return mode
    return mode.order


def spmv(A: DeviceCsr, v, mode: KernelMode | int | None = None) -> np.ndarray:
    """y = A v (kernels.hpp:348-366); host arrays in, host array out."""
    x = _aos(v, "spmv", A.K)
    y = np.empty((A.nrows, A.K))
    A.ctx.check(lib().mpsg_spmv(A.ctx.h, A.h, _order(mode), x.shape[0], _p(x), _p(y)))
    return y


def spmv_complex(A: DeviceCsr, v_re, v_im, mode: KernelMode | int | None = None):
    """(y_re, y_im) = A v (kernels.hpp:399-416)."""
    xr, xi = _aos(v_re, "spmv_complex", A.K), _aos(v_im, "spmv_complex", A.K)
    if xr.shape[0] != xi.shape[0]:
        raise ValueError("spmv_complex: re/im vector length mismatch")
    yr, yi = np.empty((A.nrows, A.K)), np.empty((A.nrows, A.K))
    A.ctx.check(lib().mpsg_spmv_complex(A.ctx.h, A.h, _order(mode), xr.shape[0], _p(xr), _p(xi), _p(yr),
                                        _p(yi)))
    return yr, yi


def _threads(mode) -> int:
    return max(1, int(getattr(mode, "threads", 1) or 1))


def sptmv(A: DeviceCsr, v, mode: KernelMode | int | None = None) -> np.ndarray:
    """y = A^T v (kernels.hpp:368-394).  The exact orders equal the reference
    sptmv at ``mode.threads`` OpenMP threads (its per-thread accumulators are
    merged in thread order, so the bits depend on the thread count).  Needs
    ``DeviceCsr(..., transpose=True)``."""
    x = _aos(v, "sptmv", A.K)
    y = np.empty((A.ncols, A.K))
    A.ctx.check(lib().mpsg_sptmv_ex(A.ctx.h, A.h, _order(mode), _threads(mode), x.shape[0], _p(x), _p(y)))
    return y


def sptmv_complex(A: DeviceCsr, v_re, v_im, mode: KernelMode | int | None = None, conjugate: bool = False):
    """(y_re, y_im) = A^T v, or the adjoint A^H v with ``conjugate`` (kernels.hpp:419-441)."""
    xr, xi = _aos(v_re, "sptmv_complex", A.K), _aos(v_im, "sptmv_complex", A.K)
    if xr.shape[0] != xi.shape[0]:
        raise ValueError("sptmv_complex: re/im vector length mismatch")
    yr, yi = np.empty((A.ncols, A.K)), np.empty((A.ncols, A.K))
    A.ctx.check(lib().mpsg_sptmv_complex_ex(A.ctx.h, A.h, _order(mode), _threads(mode), 1 if conjugate else 0,
                                            xr.shape[0], _p(xr), _p(xi), _p(yr), _p(yi)))
    return yr, yi


def sptmv_dev(A: DeviceCsr, d_v: int, d_y: int, order: int = ORDER_LANE4, stream: int | None = None):
    A.ctx.check(lib().mpsg_sptmv_dev(A.ctx.h, A.h, order, d_v, d_y, stream))


def sptmv_complex_dev(A: DeviceCsr, d_vr: int, d_vi: int, d_yr: int, d_yi: int, order: int = ORDER_LANE4,
                      conjugate: bool = False, stream: int | None = None):
    A.ctx.check(lib().mpsg_sptmv_complex_dev(A.ctx.h, A.h, order, 1 if conjugate else 0, d_vr, d_vi, d_yr, d_yi,
                                             stream))


def spmv_dev(A: DeviceCsr, d_x: int, d_y: int, order: int = ORDER_LANE4, stream: int | None = None):
    """Device-pointer SpMV, asynchronous on ``stream`` (a cudaStream_t as int)."""
    A.ctx.check(lib().mpsg_spmv_dev(A.ctx.h, A.h, order, d_x, d_y, stream))


def spmv_complex_dev(A: DeviceCsr, d_xr: int, d_xi: int, d_yr: int, d_yi: int, order: int = ORDER_LANE4,
                     stream: int | None = None):
    A.ctx.check(lib().mpsg_spmv_complex_dev(A.ctx.h, A.h, order, d_xr, d_xi, d_yr, d_yi, stream))


# --------------------------------------------------------------------------- solver
class SolverStatus(enum.IntEnum):  # krylov.hpp:46
    Converged = 0
    MaxIterations = 1
    Breakdown = 2
    Diverged = 3


class KrylovMethod(enum.IntEnum):  # krylov.hpp:24
    CG = 0
    BiCG = 1
    CGS = 2
    BiCGSTAB = 3
    GPBiCG = 4

    def __str__(self):  # to_string (krylov.hpp:26-35)
        return ("cg", "bicg", "cgs", "bicgstab", "gpbicg")[int(self)]


def parse_method(s: str) -> Optional[KrylovMethod]:  # krylov.hpp:37-44
    return {"cg": KrylovMethod.CG, "bicg": KrylovMethod.BiCG, "cgs": KrylovMethod.CGS,
            "bicgstab": KrylovMethod.BiCGSTAB, "gpbicg": KrylovMethod.GPBiCG}.get(s)


DOT_TREE, DOT_SEQUENTIAL = 0, 1


@dataclass
class SolverConfig:  # krylov.hpp:58-75
    method: KrylovMethod = KrylovMethod.BiCGSTAB
    rel_tol: float = 1e-13
    abs_tol: float = 1e-99
    max_iters: int = 10000
    threads: int = 1
    lanes_enabled: bool = True
    fast: bool = False
    x0: Sequence[float] | None = None
    check_every: int = 32
    use_graph: bool = True
    # reference dot order (one device thread per dot, krylov.hpp:122-128): with
    # an exact SpMV order the device solve reproduces the reference's bits
    exact_dots: bool = False
    # CG iteration form (mpsg_cg_variant): 0 auto (the reference's two-reduction
    # iteration on one GPU, the one-reduction Chronopoulos-Gear form when sharded
    # over several ranks), 1 classic, 2 one reduction per iteration
    cg_variant: int = 0

    def validate(self):
        if not (self.rel_tol > 0.0) or not (self.abs_tol > 0.0):
            raise ValueError("solver: tolerances must be positive")
        if self.max_iters < 1:
            raise ValueError("solver: max_iters must be at least 1")
        if self.threads < 1:
            raise ValueError("solver: threads must be at least 1")
        if self.cg_variant not in (0, 1, 2):
            raise ValueError("solver: cg_variant must be 0 (auto), 1 (classic) or 2 (one reduction)")


@dataclass
class SolverReport:  # krylov.hpp:77-88
    status: SolverStatus = SolverStatus.MaxIterations
    converged: bool = False
    detail: str = ""
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    rhs_norm: float = 0.0
    final_recurrence_residual: float = 0.0
    final_true_residual: float = 0.0
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    device_seconds: float = 0.0  # iteration loop timed with CUDA events (not in the reference)


@dataclass
class SolveResult:  # krylov.hpp:90-94
    x: np.ndarray
    report: SolverReport


@dataclass
class CsrOperator:
    """krylov.hpp:101-120: the matrix side of a solve."""

    matrix: DeviceCsr
    threads: int = 1
    lanes_enabled: bool = True
    fast: bool = False

    def rows(self) -> int:
        return self.matrix.nrows

    def cols(self) -> int:
        return self.matrix.ncols

    def mode(self) -> KernelMode:
        return KernelMode(self.threads, self.lanes_enabled, self.fast)

    def apply(self, x):
        return spmv(self.matrix, x, self.mode())

    def apply_transposed(self, x):
        return sptmv(self.matrix, x, self.mode())


def solve_cg(op: CsrOperator, b, cfg: SolverConfig | None = None) -> SolveResult:
    """Device-resident CG (krylov.hpp:238-281)."""
    cfg = cfg or SolverConfig()
    cfg.validate()
    A = op.matrix
    bb = _aos(b, "solver", A.K)
    if op.rows() != op.cols():
        raise ValueError(f"solver: operator must be square, got {op.rows()}x{op.cols()}")
    if bb.shape[0] != op.cols():
        raise ValueError("solver: rhs length does not match the operator")
    x0 = None
    if cfg.x0 is not None and len(cfg.x0) > 0:
        if len(cfg.x0) != bb.shape[0]:
            raise ValueError("solver: x0 length does not match the rhs")
        x0 = np.zeros_like(bb)
        x0[:, 0] = np.asarray(cfg.x0, dtype=np.float64)  # scalar_like (krylov.hpp:178)
    c = _CgConfig(cfg.rel_tol, cfg.abs_tol, cfg.max_iters, cfg.check_every, 1 if cfg.use_graph else 0,
                  int(cfg.cg_variant), 0)
    rep = _CgReport()
    x = np.empty_like(bb)
    hist = np.empty(cfg.max_iters + 1)
    order = ORDER_FAST if (cfg.fast or op.fast) else (ORDER_LANE4 if (cfg.lanes_enabled and op.lanes_enabled)
                                                       else ORDER_SCALAR)
    A.ctx.check(lib().mpsg_cg(A.ctx.h, A.h, order, bb.shape[0], _p(bb), _p(x0), ctypes.byref(c), _p(x),
                              _p(hist), len(hist), ctypes.byref(rep)))
    report = SolverReport(
        status=SolverStatus(rep.status), converged=bool(rep.converged), detail=rep.detail.decode(),
        iterations=int(rep.iterations), residual_history=hist[: rep.history_len].tolist(),
        rhs_norm=rep.rhs_norm, final_recurrence_residual=rep.final_recurrence_residual,
        final_true_residual=rep.final_true_residual, setup_seconds=rep.setup_seconds,
        solve_seconds=rep.solve_seconds, device_seconds=rep.device_seconds)
    return SolveResult(x, report)


def _solve_method(op: CsrOperator, b, cfg: SolverConfig, method) -> SolveResult:
    cfg.validate()
    A = op.matrix
    bb = _aos(b, "solver", A.K)
    if op.rows() != op.cols():
        raise ValueError(f"solver: operator must be square, got {op.rows()}x{op.cols()}")
    if bb.shape[0] != op.cols():
        raise ValueError("solver: rhs length does not match the operator")
    x0 = None
    if cfg.x0 is not None and len(cfg.x0) > 0:
        if len(cfg.x0) != bb.shape[0]:
            raise ValueError("solver: x0 length does not match the rhs")
        x0 = np.zeros_like(bb)
        x0[:, 0] = np.asarray(cfg.x0, dtype=np.float64)  # scalar_like (krylov.hpp:178)
    c = _SolverConfig(int(method), max(op.threads, 1), cfg.rel_tol, cfg.abs_tol, cfg.max_iters,
                      cfg.check_every, 1 if cfg.use_graph else 0,
                      DOT_SEQUENTIAL if cfg.exact_dots else DOT_TREE, 0)
    rep = _CgReport()
    x = np.empty_like(bb)
    hist = np.empty(cfg.max_iters + 1)
    order = ORDER_FAST if (cfg.fast or op.fast) else (ORDER_LANE4 if (cfg.lanes_enabled and op.lanes_enabled)
                                                       else ORDER_SCALAR)
    A.ctx.check(lib().mpsg_solve(A.ctx.h, A.h, order, bb.shape[0], _p(bb), _p(x0), ctypes.byref(c), _p(x),
                                 _p(hist), len(hist), ctypes.byref(rep)))
    report = SolverReport(
        status=SolverStatus(rep.status), converged=bool(rep.converged), detail=rep.detail.decode(),
        iterations=int(rep.iterations), residual_history=hist[: rep.history_len].tolist(),
        rhs_norm=rep.rhs_norm, final_recurrence_residual=rep.final_recurrence_residual,
        final_true_residual=rep.final_true_residual, setup_seconds=rep.setup_seconds,
        solve_seconds=rep.solve_seconds, device_seconds=rep.device_seconds)
    return SolveResult(x, report)


def solve(op: CsrOperator, b, cfg: SolverConfig | None = None) -> SolveResult:
    """solve() (krylov.hpp:596-606): the device-resident Krylov method
    cfg.method (CG, BiCG, CGS, BiCGSTAB, GPBiCG).  BiCG needs a matrix
    uploaded with ``transpose=True``."""
    cfg = cfg or SolverConfig()
    return _solve_method(op, b, cfg, cfg.method)


def solve_bicg(op: CsrOperator, b, cfg: SolverConfig | None = None) -> SolveResult:  # krylov.hpp:283
    return _solve_method(op, b, cfg or SolverConfig(), KrylovMethod.BiCG)


def solve_cgs(op: CsrOperator, b, cfg: SolverConfig | None = None) -> SolveResult:  # krylov.hpp:339
    return _solve_method(op, b, cfg or SolverConfig(), KrylovMethod.CGS)


def solve_bicgstab(op: CsrOperator, b, cfg: SolverConfig | None = None) -> SolveResult:  # krylov.hpp:398
    return _solve_method(op, b, cfg or SolverConfig(), KrylovMethod.BiCGSTAB)


def solve_gpbicg(op: CsrOperator, b, cfg: SolverConfig | None = None) -> SolveResult:  # krylov.hpp:478
    return _solve_method(op, b, cfg or SolverConfig(), KrylovMethod.GPBiCG)


# --------------------------------------------------------------------------- multi-GPU
NCCL_ID_BYTES = 128


class Comm:
    """One rank of a row-sharded group (mpsg_comm over NCCL).  ``unique_id``
    comes from ``Comm.unique_id()`` on one rank, broadcast by the caller (e.g.
    torch.distributed.broadcast_object_list)."""

    def __init__(self, ctx: Context, nranks: int = 1, rank: int = 0, unique_id: bytes | None = None):
        self.ctx, self.nranks, self.rank = ctx, nranks, rank
        buf = None
        if unique_id is not None:
            buf = ctypes.create_string_buffer(bytes(unique_id), NCCL_ID_BYTES)
        h = _P()
        ctx.check(lib().mpsg_comm_create(ctx.h, nranks, rank, buf, ctypes.byref(h)))
        self.h = h

    @classmethod
    def local_group(cls, ctxs):
        """One process, one host thread per rank: comms for len(ctxs) ranks
        whose collectives are event-ordered device/peer copies (no NCCL)."""
        n = len(ctxs)
        arr = (_P * n)(*[c.h for c in ctxs])
        outs = (_P * n)()
        rc = lib().mpsg_comm_create_local(arr, n, outs)
        if rc != E_OK:
            raise MpsgError(rc, "mpsg_comm_create_local failed")
        comms = []
        for r in range(n):
            c = cls.__new__(cls)
            c.ctx, c.nranks, c.rank, c.h = ctxs[r], n, r, _P(outs[r])
            comms.append(c)
        return comms

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
        rc = lib().mpsg_comm_unique_id(buf)
        if rc != E_OK:
            raise MpsgError(rc, "mpsg_comm_unique_id failed (libnccl.so.2 not loadable?)")
        return buf.raw

    def close(self):
        if getattr(self, "h", None):
            lib().mpsg_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_rows(A, row_begin: int, row_end: int):
    """Rows [row_begin, row_end) of a reference-layout CSR, indptr rebased,
    global column indices kept (host helper for DistCsr)."""
    from types import SimpleNamespace

    ip = np.asarray(A.indptr, dtype=np.int64)
    lo, hi = int(ip[row_begin]), int(ip[row_end])
    return SimpleNamespace(nrows=row_end - row_begin, ncols=int(A.ncols), indptr=ip[row_begin:row_end + 1] - lo,
                           indices=np.asarray(A.indices, dtype=np.int64)[lo:hi],
                           planes=np.asarray(A.planes)[:, lo:hi])


class DistCsr:
    """This rank's row block of a square matrix (mpsg_dcsr).  Collective."""

    def __init__(self, comm: Comm, A_local, K: int, nglobal: int, row_begin: int, row_end: int,
                 is_complex: bool = False):
        self.comm, self.K, self.is_complex = comm, K, bool(is_complex)
        self.nglobal, self.row_begin, self.row_end = int(nglobal), int(row_begin), int(row_end)
        indptr = np.ascontiguousarray(A_local.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(A_local.indices, dtype=np.int64)
        nplanes = 2 * K if is_complex else K
        plist = [np.ascontiguousarray(np.asarray(A_local.planes)[j], dtype=np.float64) for j in range(nplanes)]
        parr = (_P * nplanes)(*[p.ctypes.data for p in plist])
        h = _P()
        comm.ctx.check(lib().mpsg_dcsr_upload(comm.h, K, 1 if is_complex else 0, self.nglobal, self.row_begin,
                                              self.row_end, _p(indptr), _p(indices), parr, ctypes.byref(h)))
        self.h = h

    @classmethod
    def from_global(cls, comm: Comm, A, K: int, is_complex: bool = False, bounds=None):
        """Shard a full host matrix by the reference's equal-nnz rule (or ``bounds``)."""
        if bounds is None:
            bounds = partition_rows(A.indptr, int(A.nrows), comm.nranks)
        b, e = int(bounds[comm.rank]), int(bounds[comm.rank + 1])
        return cls(comm, shard_rows(A, b, e), K, int(A.nrows), b, e, is_complex)

    def info(self):
        b = np.empty(self.comm.nranks + 1, dtype=np.int64)
        halo = _i64()
        self.comm.ctx.check(lib().mpsg_dcsr_info(self.h, _p(b), ctypes.byref(halo)))
        return b, int(halo.value)

    def interior_rows(self) -> int:
        """Rows computed while the x halo moves (columns all in this rank's block)."""
        v = _i64()
        self.comm.ctx.check(lib().mpsg_dcsr_interior_rows(self.h, ctypes.byref(v)))
        return int(v.value)

    def close(self):
        if getattr(self, "h", None):
            lib().mpsg_dcsr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dspmv(A: DistCsr, x_local, mode: KernelMode | int | None = None) -> np.ndarray:
    """y_local = (A x)[this rank's rows]; x_local is this rank's block.  Collective."""
    x = _aos(x_local, "spmv", A.K)
    if x.shape[0] != A.row_end - A.row_begin:
        raise ValueError(f"spmv: vector length {x.shape[0]} does not match the row block "
                         f"{A.row_end - A.row_begin}")
    y = np.empty((A.row_end - A.row_begin, A.K))
    A.comm.ctx.check(lib().mpsg_dspmv(A.h, _order(mode), _p(x), _p(y)))
    return y


def dspmv_dev(A: DistCsr, d_x: int, d_y: int, order: int = ORDER_LANE4, stream: int | None = None):
    A.comm.ctx.check(lib().mpsg_dspmv_dev(A.h, order, d_x, d_y, stream))


def dspmv_complex_dev(A: DistCsr, d_xr: int, d_xi: int, d_yr: int, d_yi: int, order: int = ORDER_LANE4,
                      stream: int | None = None):
    A.comm.ctx.check(lib().mpsg_dspmv_complex_dev(A.h, order, d_xr, d_xi, d_yr, d_yi, stream))


def dsolve_cg(A: DistCsr, b_local, cfg: SolverConfig | None = None) -> SolveResult:
    """Row-sharded device CG; b_local / result x are this rank's blocks.  Collective."""
    cfg = cfg or SolverConfig()
    cfg.validate()
    bb = _aos(b_local, "solver", A.K)
    if bb.shape[0] != A.row_end - A.row_begin:
        raise ValueError("solver: rhs length does not match the operator")
    x0 = None
    if cfg.x0 is not None and len(cfg.x0) > 0:
        if len(cfg.x0) != A.nglobal:
            raise ValueError("solver: x0 length does not match the rhs")
        x0 = np.zeros_like(bb)
        x0[:, 0] = np.asarray(cfg.x0, dtype=np.float64)[A.row_begin:A.row_end]
    c = _CgConfig(cfg.rel_tol, cfg.abs_tol, cfg.max_iters, cfg.check_every, 1 if cfg.use_graph else 0,
                  int(cfg.cg_variant), 0)
    rep = _CgReport()
    x = np.empty_like(bb)
    hist = np.empty(cfg.max_iters + 1)
    order = ORDER_FAST if cfg.fast else (ORDER_LANE4 if cfg.lanes_enabled else ORDER_SCALAR)
    A.comm.ctx.check(lib().mpsg_dcg(A.h, order, _p(bb), _p(x0), ctypes.byref(c), _p(x), _p(hist), len(hist),
                                    ctypes.byref(rep)))
    report = SolverReport(
        status=SolverStatus(rep.status), converged=bool(rep.converged), detail=rep.detail.decode(),
        iterations=int(rep.iterations), residual_history=hist[: rep.history_len].tolist(),
        rhs_norm=rep.rhs_norm, final_recurrence_residual=rep.final_recurrence_residual,
        final_true_residual=rep.final_true_residual, setup_seconds=rep.setup_seconds,
        solve_seconds=rep.solve_seconds, device_seconds=rep.device_seconds)
    return SolveResult(x, report)


def dsolve(A: DistCsr, b_local, cfg: SolverConfig | None = None) -> SolveResult:
    """Row-sharded device solve() (CG, CGS, BiCGSTAB, GPBiCG; cfg.method);
    b_local / result x are this rank's blocks, the report is identical on
    every rank.  Collective."""
    cfg = cfg or SolverConfig()
    cfg.validate()
    bb = _aos(b_local, "solver", A.K)
    if bb.shape[0] != A.row_end - A.row_begin:
        raise ValueError("solver: rhs length does not match the operator")
    x0 = None
    if cfg.x0 is not None and len(cfg.x0) > 0:
        if len(cfg.x0) != A.nglobal:
            raise ValueError("solver: x0 length does not match the rhs")
        x0 = np.zeros_like(bb)
        x0[:, 0] = np.asarray(cfg.x0, dtype=np.float64)[A.row_begin:A.row_end]
    c = _SolverConfig(int(cfg.method), max(cfg.threads, 1), cfg.rel_tol, cfg.abs_tol, cfg.max_iters,
                      cfg.check_every, 1 if cfg.use_graph else 0, DOT_SEQUENTIAL if cfg.exact_dots else DOT_TREE, 0)
    rep = _CgReport()
    x = np.empty_like(bb)
    hist = np.empty(cfg.max_iters + 1)
    order = ORDER_FAST if cfg.fast else (ORDER_LANE4 if cfg.lanes_enabled else ORDER_SCALAR)
    A.comm.ctx.check(lib().mpsg_dsolve(A.h, order, _p(bb), _p(x0), ctypes.byref(c), _p(x), _p(hist), len(hist),
                                       ctypes.byref(rep)))
    report = SolverReport(
        status=SolverStatus(rep.status), converged=bool(rep.converged), detail=rep.detail.decode(),
        iterations=int(rep.iterations), residual_history=hist[: rep.history_len].tolist(),
        rhs_norm=rep.rhs_norm, final_recurrence_residual=rep.final_recurrence_residual,
        final_true_residual=rep.final_true_residual, setup_seconds=rep.setup_seconds,
        solve_seconds=rep.solve_seconds, device_seconds=rep.device_seconds)
    return SolveResult(x, report)


def halo_plan(nranks: int, rank: int, bounds, need):
    """Host-only halo plan (mpsg_halo_plan): returns (send, recv), each [nranks, 2]."""
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    nd = np.ascontiguousarray(need, dtype=np.int64).reshape(-1)
    send = np.empty(2 * nranks, dtype=np.int64)
    recv = np.empty(2 * nranks, dtype=np.int64)
    rc = lib().mpsg_halo_plan(nranks, rank, _p(b), _p(nd), _p(send), _p(recv))
    if rc != E_OK:
        raise ValueError("halo_plan: bad arguments")
    return send.reshape(nranks, 2), recv.reshape(nranks, 2)


def need_interval(A_local, row_begin: int, row_end: int):
    """Column interval a row block reads (its own block included)."""
    idx = np.asarray(A_local.indices)
    lo = min(row_begin, int(idx.min())) if len(idx) else row_begin
    hi = max(row_end, int(idx.max()) + 1) if len(idx) else row_end
    return lo, hi


# --------------------------------------------------------------------------- host utilities
def partition_rows(indptr, nrows: int, parts: int) -> np.ndarray:
    """nnz-balanced contiguous row bounds (kernels.hpp:63-80)."""
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    out = np.empty(parts + 1, dtype=np.int64)
    rc = lib().mpsg_partition_rows(_p(ip), nrows, parts, _p(out))
    if rc != E_OK:
        raise ValueError("partition_rows: bad arguments")
    return out


def checksum(v) -> int:
    a = _aos(v, "checksum")
    return int(lib().mpsg_checksum(a.shape[1], a.shape[0], _p(a)))


def checksum_complex(re, im) -> int:
    r, i = _aos(re), _aos(im)
    return int(lib().mpsg_checksum_complex(r.shape[1], r.shape[0], _p(r), _p(i)))


def measure_fp64_peak(ctx: Optional[Context] = None) -> float:
    """fp64 instructions per second (DFMA throughput) on the context's GPU."""
    ctx = ctx or default_context()
    v = _f64()
    ctx.check(lib().mpsg_measure_fp64_peak(ctx.h, ctypes.byref(v)))
    return float(v.value)


MC_OPS = {"add": 0, "mul": 1, "mul_d": 2, "sub": 3, "div": 4, "sqrt": 5}


def mc_op_dev(ctx: Context, op: str, K: int, n: int, d_a: int, d_b: int, d_out: int):
    """Batched device MC op on AoS device arrays (asynchronous on the context stream)."""
    ctx.check(lib().mpsg_mc_op_dev(ctx.h, MC_OPS[op], K, n, d_a, d_b, d_out))


def make_vector(ctx: Context, K: int, n: int, complex: bool = False):
    """The reference harness's input vector (bench.hpp:78-111): v_j = sqrt(2) j,
    or (re, im) of sqrt(2 + 3i) j, computed on the device with the reference's ops."""
    re = np.empty((n, K))
    im = np.empty((n, K)) if complex else None
    ctx.check(lib().mpsg_make_vector(ctx.h, K, n, _p(re), _p(im)))
    return (re, im) if complex else re


def version() -> str:
    return lib().mpsg_version().decode()
