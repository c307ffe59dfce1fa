"""The FAST order's fused product-accumulate (mc_arith.cuh fma_acc / fma_fast:
one renormalisation per nonzero, the accumulator kept by the renorm's backward
sweep) against the north-star componentwise bound
|y - y_ref| <= 4 rowlen u sum|a||x| (u = 2^-104 / 2^-156 / 2^-208), row by row,
on inputs chosen to stress it: power-law long rows (the long-row kernel's
chunked chains), a 2^+-60 exponent spread, exact pairwise cancellation, Mixed
mode, complex.  The worst ratio must stay well inside the bound (the measured
worst is 0.18 for TD and 0.15 for QD, both on length-1 rows of the power-law
matrix, where the bound is tightest and the difference is the reference's own
product truncation; tools/fused_adversarial.py)."""
import numpy as np
import pytest

import oracle as O
import paper_2412_17510_b200 as M
import synth
from tests.util import bound_ok, mixed_of

pytestmark = pytest.mark.gpu

MARGIN = 0.25  # worst |error| / bound allowed here (the contract is 1.0)


@pytest.fixture(scope="module")
def ctx():
    c = M.Context(0)
    yield c
    c.close()


def _check(A, x, y, K, mixed=False):
    ok, worst = bound_ok(A, x, y, O.spmv(A, x, 0, mixed=mixed), K)
    assert ok and worst <= MARGIN, worst
    return worst


@pytest.mark.parametrize("K", [2, 3, 4])
def test_fast_power_law_long_rows(ctx, K):
    c = M.Context(0)
    c.set_layout(long_threshold=64, sigma=1024, fast_chunk=256)  # many long rows, several chunks each
    A = synth.config_matrix(4, K, 20000, 6000.0, 1.8)
    x = synth.config_vector(4, A.nrows, K)
    _check(A, x, M.spmv(M.DeviceCsr(A, K, ctx=c), x, M.ORDER_FAST), K)
    c.close()


@pytest.mark.parametrize("K", [2, 3, 4])
def test_fast_wide_exponent_range(ctx, K):
    rng = np.random.default_rng(K)
    A = synth.config_matrix(2, K, 20000, 40.0)
    A.planes *= np.exp2(rng.integers(-60, 61, A.planes.shape[1])).astype(float)[None, :]
    x = synth.config_vector(2, A.nrows, K) * np.exp2(rng.integers(-60, 61, A.nrows)).astype(float)[:, None]
    _check(A, x, M.spmv(M.DeviceCsr(A, K, ctx=ctx), x, M.ORDER_FAST), K)


@pytest.mark.parametrize("K", [2, 3, 4])
def test_fast_exact_cancellation(ctx, K):
    """Adjacent a / -a pairs times a CONSTANT x, so the running accumulator
    really cancels: exactly (whole pairs), down to a level-1 residue (the
    pair agrees in its leading component only) and down to a level-2 residue
    (leading two agree).  The fused accumulate then runs with s0 ~ 0 and its
    non-canonical accumulator fed back in -- the case where the level-wise
    quick-two-sums see |h| > |s0|."""
    rng = np.random.default_rng(100 + K)
    A = synth.config_matrix(2, K, 20000, 40.0)
    P = A.planes
    m = P[:, 1::2].shape[1]
    P[:, 1::2] = -P[:, 0::2][:, :m]
    kind = rng.integers(0, 3, m)  # 0: exact, 1: level-1 residue, 2: level-2 residue
    for lev in (1, 2):
        if lev >= K:
            continue
        sel = np.nonzero(kind == lev)[0]
        fresh = synth.vector(synth.VAL_NORMAL, len(sel), K, seed=7 + lev).T  # (K, len)
        for j in range(lev, K):
            P[j, 1 + 2 * sel] = fresh[j] * np.abs(P[lev - 1, 1 + 2 * sel]) * 2.0 ** (-53 * (j - lev + 1))
    x1 = synth.config_vector(2, 1, K)[0]
    x = np.tile(x1, (A.nrows, 1))
    w = _check(A, x, M.spmv(M.DeviceCsr(A, K, ctx=ctx), x, M.ORDER_FAST), K)
    assert np.isfinite(w)


@pytest.mark.parametrize("K", [3, 4])
def test_fast_mixed_mode(ctx, K):
    A = mixed_of(synth.config_matrix(2, K, 20000, 40.0))
    x = synth.config_vector(2, A.nrows, K)
    _check(A, x, M.spmv(M.DeviceCsr(A, K, ctx=ctx, mixed=True), x, M.ORDER_FAST), K, mixed=True)


@pytest.mark.parametrize("K", [3, 4])
def test_fast_complex(ctx, K):
    A = synth.config_matrix(3, K, 4000, 24.0)
    xr, xi = synth.config_vector(3, A.nrows, K)
    yr, yi = M.spmv_complex(M.DeviceCsr(A, K, True, ctx=ctx), xr, xi, M.ORDER_FAST)
    rr, ri = O.spmv_complex(A, xr, xi, 0)
    s = O.abs_rowsum(A, A.planes[0], xr) + O.abs_rowsum(A, A.planes[K], xi)
    s = s + O.abs_rowsum(A, A.planes[0], xi) + O.abs_rowsum(A, A.planes[K], xr)
    for y, ref in ((yr, rr), (yi, ri)):
        ok, worst = bound_ok(A, xr, y, ref, K, extra=s)
        assert ok and worst <= MARGIN, worst


def test_fast_output_is_canonical(ctx):
    """Stored FAST results are renormalised (the per-row canon()): each lower
    component is at most half an ulp of the one above."""
    K = 4
    A = synth.config_matrix(2, K, 20000, 40.0)
    x = synth.config_vector(2, A.nrows, K)
    y = M.spmv(M.DeviceCsr(A, K, ctx=ctx), x, M.ORDER_FAST)
    for j in range(K - 1):
        hi, lo = y[:, j], y[:, j + 1]
        nz = hi != 0
        assert np.all(np.abs(lo[nz]) <= np.spacing(np.abs(hi[nz])) / 2 * (1 + 1e-12))
