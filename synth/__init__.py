"""Seeded synthetic inputs for the five BASELINE.json configs (see mpsgen.c).

Shared by the parity tests and bench.py.  Matrices come back in the
reference's CSR form (int64 ``indptr``/``indices``, sparse.hpp:69-78) with the
values as K component planes ``[K, nnz]`` (CsrValues SoA, sparse.hpp:47-67);
complex matrices carry ``[2K, nnz]`` (re planes then im planes).  Vectors are
AoS ``[n, K]`` float64, the memory image of ``std::vector<MultiComponent<K>>``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libmpsgen.so")

VAL_UNIFORM, VAL_NORMAL, VAL_UNIFORM0 = 0, 1, 2

# Full BASELINE.json sizes: (p1, p2, p3) per config.
FULL = {
    1: (512, 0.0, 0.0),  # 2D Laplacian 512x512
    2: (1_000_000, 32.0, 0.0),  # Poisson(32) random, n = 1e6
    3: (500_000, 32.0, 0.0),  # banded, half-bandwidth 32, complex
    4: (4_000_000, 50000.0, 1.8),  # Zipf(1.8) clipped to [1, 50000]
    5: (128, 0.0, 0.0),  # 3D 7-point Laplacian 128^3
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run `make -C synth` (or __graft_entry__.build())")
        L = ctypes.CDLL(_LIB)
        i64, f64, u64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int
        P = ctypes.c_void_p
        L.gen_nrows.argtypes = [i32, i64]
        L.gen_nrows.restype = i64
        L.gen_indptr.argtypes = [i32, i64, f64, f64, u64, P]
        L.gen_indptr.restype = i64
        L.gen_fill.argtypes = [i32, i64, f64, u64, i32, P, P, P]
        L.gen_fill.restype = None
        L.gen_vector.argtypes = [i32, i64, u64, i32, i32, P]
        L.gen_vector.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class HostCsr:
    """Host CSR in the reference's layout (int64 indices, SoA value planes)."""

    nrows: int
    ncols: int
    indptr: np.ndarray  # int64 [nrows+1]
    indices: np.ndarray  # int64 [nnz]
    planes: np.ndarray  # float64 [K or 2K, nnz]
    K: int
    is_complex: bool = False

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    @property
    def re(self) -> np.ndarray:
        return self.planes[: self.K]

    @property
    def im(self) -> np.ndarray:
        return self.planes[self.K :]


def config_matrix(cfg: int, K: int, p1=None, p2=None, p3=None, seed: int = 0) -> HostCsr:
    fp1, fp2, fp3 = FULL[cfg]
    p1 = fp1 if p1 is None else p1
    p2 = fp2 if p2 is None else p2
    p3 = fp3 if p3 is None else p3
    L = lib()
    n = L.gen_nrows(cfg, p1)
    indptr = np.empty(n + 1, dtype=np.int64)
    nnz = L.gen_indptr(cfg, p1, float(p2), float(p3), seed, _ptr(indptr))
    indices = np.empty(nnz, dtype=np.int64)
    nplanes = 2 * K if cfg == 3 else K
    planes = np.empty((nplanes, nnz), dtype=np.float64)
    L.gen_fill(cfg, p1, float(p2), seed, K, _ptr(indptr), _ptr(indices), _ptr(planes))
    return HostCsr(n, n, indptr, indices, planes, K, cfg == 3)


def vector(style: int, n: int, K: int, seed: int = 0, imag: bool = False) -> np.ndarray:
    out = np.empty((n, K), dtype=np.float64)
    lib().gen_vector(style, n, seed, K, 1 if imag else 0, _ptr(out))
    return out


def config_vector(cfg: int, n: int, K: int, seed: int = 1):
    """x for a config: U-style for 1/4, N-style for 2/3 (complex pair for 3),
    U with zero tail (x_true) for 5."""
    if cfg in (1, 4):
        return vector(VAL_UNIFORM, n, K, seed)
    if cfg == 2:
        return vector(VAL_NORMAL, n, K, seed)
    if cfg == 3:
        return vector(VAL_NORMAL, n, K, seed), vector(VAL_NORMAL, n, K, seed, imag=True)
    if cfg == 5:
        return vector(VAL_UNIFORM0, n, K, seed)
    raise ValueError(cfg)
