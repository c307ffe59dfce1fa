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


def krylov_system(n, K, seed=0, symmetric=False, density=0.1, dominance=1.0):
    """Seeded diagonally dominant n x n system with full-width K-component
    values (like the reference's random_diag_dominant, tests/support/
    fixtures.hpp) and a right-hand side b; test-side generator."""
    import synth

    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    if symmetric:
        mask = np.triu(mask, 1)
        mask = mask | mask.T
    np.fill_diagonal(mask, True)
    rows = [np.nonzero(mask[i])[0].tolist() for i in range(n)]
    A = csr(n, n, rows, K, seed=seed + 1)
    hi = A.planes[0]
    if symmetric:  # mirror the values of the upper triangle
        pos = {}
        for i in range(n):
            for k in range(A.indptr[i], A.indptr[i + 1]):
                pos[(i, int(A.indices[k]))] = k
        for (i, j), k in pos.items():
            if j < i:
                A.planes[:, k] = A.planes[:, pos[(j, i)]]
    for i in range(n):
        lo, hi_ = A.indptr[i], A.indptr[i + 1]
        off = [k for k in range(lo, hi_) if A.indices[k] != i]
        d = [k for k in range(lo, hi_) if A.indices[k] == i][0]
        A.planes[:, d] = 0.0
        A.planes[0, d] = float(np.sum(np.abs(hi[off]))) * dominance + 1.0 + rng.random()
    b = synth.vector(synth.VAL_NORMAL, n, K, seed=seed + 2)
    return A, b


# small integer systems that drive each solver into one of its breakdown exits
# (found by a seeded search with the oracle; reference detail texts)
BREAKDOWN_CASES = [
    ("bicg", [[1, -2], [-1, 0]], [0, -2], "bicg: <p~, Ap> vanished"),
    ("bicg", [[1, 0], [2, 2]], [-1, 0], "bicg: <r~, r> vanished"),
    ("cgs", [[1, -2], [-1, 0]], [0, -2], "cgs: <r~, Ap> vanished"),
    ("cgs", [[1, 0], [2, 2]], [-1, 0], "cgs: <r~, r> vanished"),
    ("bicgstab", [[1, -2], [-1, 0]], [0, -2], "bicgstab: <r~, Ap> vanished"),
    ("bicgstab", [[2, 2, 0], [-2, -2, 0], [-2, -2, 1]], [-1, -2, 2], "bicgstab: <r~, r> vanished"),
    ("bicgstab", [[1, 1], [2, 2]], [2, 2], "bicgstab: <t, t> vanished"),
    ("bicgstab", [[0, 2], [-1, -2]], [0, -2], "bicgstab: omega vanished"),
    ("gpbicg", [[0, 2], [0, -1]], [0, 1], "gpbicg: <At, At> vanished"),
    ("gpbicg", [[1, -2], [-1, 0]], [0, -2], "gpbicg: <r~, Ap> vanished"),
    ("gpbicg", [[2, 2, -2], [1, 1, 2], [-1, 2, -1]], [2, 2, 0], "gpbicg: <r~, r> vanished"),
    ("gpbicg", [[0, 2], [-1, -2]], [0, -2], "gpbicg: zeta vanished"),
    ("gpbicg", [[1, -1], [2, -2]], [2, 1], "gpbicg: zeta/eta system is singular"),
    ("cg", [[0, 1], [-1, 0]], [1, 1], "cg: <p, Ap> vanished"),
]


def dense_system(M, bvec, K=2):
    """Integer dense matrix / rhs -> K-component CSR + AoS rhs (zero tails)."""
    M = np.asarray(M, float)
    n = M.shape[0]
    rows = [[j for j in range(n) if M[i, j] != 0] for i in range(n)]
    vals = np.array([M[i, j] for i in range(n) for j in rows[i]])
    planes = np.zeros((K, len(vals)))
    planes[0] = vals
    b = np.zeros((n, K))
    b[:, 0] = bvec
    return csr(n, n, rows, K, planes=planes), b


def krylov_mixed_cases():
    """(name, A_binary64, b, method, kwargs): solve() over CsrOperator<double>
    (Mixed mode, the binary64 leading plane) with K-component vectors."""
    out = []
    for K in (2, 3, 4):
        for sym in (True, False):
            A, b = krylov_system(60, K, seed=13, symmetric=sym)
            Am = mixed_of(A)
            for m in ("cg", "bicg", "cgs", "bicgstab", "gpbicg"):
                if m == "cg" and not sym:
                    continue
                out.append((f"mixed_{'sym' if sym else 'nonsym'}_K{K}_{m}", Am, b, m, {}))
    A, b = krylov_system(60, 2, seed=13, symmetric=False)
    out.append(("mixed_nonsym_K2_bicg_t4", mixed_of(A), b, "bicg", {"threads": 4}))
    return out


def krylov_cases():
    """(name, A, b, method, kwargs) parity cases shared by the oracle golden, the
    oracle tests and the device tests."""
    out = []
    for sym in (True, False):
        for K in (2, 3, 4):
            A, b = krylov_system(60, K, seed=3, symmetric=sym)
            for m in ("cg", "bicg", "cgs", "bicgstab", "gpbicg"):
                if m == "cg" and not sym:
                    continue
                out.append((f"{'sym' if sym else 'nonsym'}_K{K}_{m}", A, b, m, {}))
    A, b = krylov_system(60, 2, seed=3, symmetric=False)
    out.append(("nonsym_K2_bicg_t3", A, b, "bicg", {"threads": 3}))
    A, b = krylov_system(40, 3, seed=5, symmetric=False, dominance=0.2)
    for m in ("bicg", "cgs", "bicgstab", "gpbicg"):
        out.append((f"weak_K3_{m}", A, b, m, {"max_iters": 300}))
    A, b = krylov_system(30, 4, seed=9, symmetric=True)
    for m in ("cg", "bicg", "cgs", "bicgstab", "gpbicg"):
        out.append((f"maxit_K4_{m}", A, b, m, {"rel_tol": 1e-60, "max_iters": 15}))
    I, bi = dense_system(np.eye(6), [0.5, -1.25, 2.0, 3.5, -0.75, 1.0])
    D, bd = dense_system(np.diag([1.0, 2.0, 4.0]), [1.0, 4.0, 16.0])
    for m in ("cg", "bicg", "cgs", "bicgstab", "gpbicg"):
        out.append((f"identity_{m}", I, bi, m, {}))
        out.append((f"x0exact_{m}", D, bd, m, {"x0": [1.0, 2.0, 4.0]}))
        out.append((f"x0_{m}", D, bd, m, {"x0": [0.5, -1.0, 3.0]}))
    for i, (m, M, bv, _) in enumerate(BREAKDOWN_CASES):
        A, b = dense_system(M, bv)
        out.append((f"breakdown{i}_{m}", A, b, m, {"max_iters": 50}))
    return out
