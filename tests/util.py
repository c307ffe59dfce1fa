"""Shared helpers for the parity tests (test-side only)."""
from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# unit roundoff per width (BASELINE.json north_star bound)
U = {2: 2.0**-104, 3: 2.0**-156, 4: 2.0**-208}

_cache = {}


def golden(name: str):
    if name not in _cache:
        _cache[name] = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return _cache[name]


def widen(m, K):
    """binary64 matrix -> K-component matrix with zero tails (convert_csr, sparse.hpp:195-207)."""
    planes = np.zeros((K, m.nnz if hasattr(m, "nnz") else len(m.indices)))
    planes[0] = np.asarray(m.planes)[0]
    return SimpleNamespace(nrows=m.nrows, ncols=m.ncols, indptr=np.asarray(m.indptr, np.int64),
                           indices=np.asarray(m.indices, np.int64), planes=planes, K=K, nnz=planes.shape[1])


def csr(nrows, ncols, rows, K, planes=None, seed=0, is_complex=False):
    """CSR from per-row column lists; random N-style values unless planes given."""
    indptr = np.zeros(nrows + 1, np.int64)
    for i, r in enumerate(rows):
        indptr[i + 1] = indptr[i] + len(r)
    indices = np.array([c for r in rows for c in r], dtype=np.int64)
    nnz = len(indices)
    if planes is None:
        import synth

        npl = 2 * K if is_complex else K
        v = synth.vector(synth.VAL_NORMAL, nnz * (2 if is_complex else 1), K, seed=seed)
        if is_complex:
            planes = np.concatenate([v[:nnz].T, v[nnz:].T], axis=0)
        else:
            planes = v.T.copy()
        assert planes.shape[0] == npl
    return SimpleNamespace(nrows=nrows, ncols=ncols, indptr=indptr, indices=indices,
                           planes=np.ascontiguousarray(planes), K=K, nnz=nnz)


def bits_equal(a, b) -> bool:
    """Bit-for-bit equality, except that any NaN equals any NaN: x86 produces the
    default negative quiet NaN (0xfff8...) for invalid operations where sm_100
    produces the canonical 0x7fff...; NaN-ness itself must match."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return bool(np.array_equal(a.view(np.uint64)[~na], b.view(np.uint64)[~nb]))


def first_mismatch(a, b):
    av = np.ascontiguousarray(a).view(np.uint64)
    bv = np.ascontiguousarray(b).view(np.uint64)
    bad = np.argwhere((av != bv) & ~(np.isnan(a) & np.isnan(b)))
    return None if len(bad) == 0 else (tuple(bad[0]), a[tuple(bad[0])[0]], b[tuple(bad[0])[0]], len(bad))


def bound_ok(A, x, y, yref, K, extra=None):
    """|y - y_ref| <= 4 * rowlen * u * sum_j |a_ij||x_j| for every row (north-star bound).
    Returns (ok, worst ratio)."""
    import oracle as O

    rowlen = np.diff(A.indptr).astype(float)
    s = O.abs_rowsum(A, A.planes[0], x) if extra is None else extra
    d = O.exact_absdiff(y, yref)
    lim = 4.0 * np.maximum(rowlen, 1.0) * U[K] * s
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(lim > 0, d / lim, np.where(d == 0, 0.0, np.inf))
    return bool(np.all(d <= lim)), float(np.max(ratio)) if len(ratio) else 0.0


def mixed_of(A, cplx=False):
    """The binary64 matrix of Mixed mode: the leading plane (re, im for complex)."""
    K = A.K
    planes = np.stack([A.planes[0], A.planes[K]]) if cplx else A.planes[:1].copy()
    return SimpleNamespace(nrows=A.nrows, ncols=A.ncols, indptr=A.indptr, indices=A.indices,
                           planes=np.ascontiguousarray(planes), K=K, nnz=A.nnz)


def transpose(A):
    """Host A^T with rows listing entries in ascending original row (transpose_csr, sparse.hpp:139-163)."""
    indptr = np.asarray(A.indptr, np.int64)
    rows = np.repeat(np.arange(A.nrows, dtype=np.int64), np.diff(indptr))
    cols = np.asarray(A.indices, np.int64)
    perm = np.lexsort((rows, cols))
    tptr = np.zeros(A.ncols + 1, np.int64)
    np.add.at(tptr, cols + 1, 1)
    tptr = np.cumsum(tptr)
    planes = np.ascontiguousarray(np.asarray(A.planes)[:, perm])
    return SimpleNamespace(nrows=A.ncols, ncols=A.nrows, indptr=tptr, indices=rows[perm], planes=planes,
                           K=getattr(A, "K", None), nnz=len(perm))
