"""FAST order at the BASELINE.json sizes the bench times (north star: "the fast
kernels must satisfy a componentwise bound against the reference").

Every row of the FAST result of each full-size config is checked against the
reference's lanes-off output (row_sum_scalar, kernels.hpp:90-99; complex
kernels.hpp:399-416) with |y - y_ref| <= 4 rowlen u sum|a_ij||x_j|,
u = 2^-104 / 2^-156 / 2^-208.  The reference output comes from the unmodified
reference (oracle/_ref/libmpsref.so, all host threads) when it was built,
else from the C restatement pinned bit-exact to it (tests/test_oracle.py).
These are the matrices and kernels `bench.py` / `bench.py --all` measure:
cfg1 DD, cfg2 TD / QD, cfg3 complex DD / QD, cfg4 DD (every row: SELL short
rows and the column-blocked long rows), cfg5 DD / QD.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2412_17510_b200 as M
import synth
from tests.util import bound_ok

pytestmark = pytest.mark.gpu

MARGIN = 0.25  # worst |error| / bound allowed (the contract is 1.0)
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def ctx():
    c = M.Context(0)
    yield c
    c.close()


def _ref_real(A, x):
    if O.ref_available():
        return O.ref_spmv(A, x, O.SCALAR, threads=THREADS)
    return O.spmv(A, x, O.SCALAR)


def _ref_complex(A, xr, xi):
    if O.ref_available():
        return O.ref_spmv_complex(A, xr, xi, O.SCALAR, threads=THREADS)
    return O.spmv_complex(A, xr, xi, O.SCALAR)


@pytest.mark.parametrize("cfg,K", [(1, 2), (2, 3), (2, 4), (4, 2), (5, 2), (5, 4)],
                         ids=["cfg1_DD", "cfg2_TD", "cfg2_QD", "cfg4_DD", "cfg5_DD", "cfg5_QD"])
def test_fast_full_size_within_bound(ctx, cfg, K):
    A = synth.config_matrix(cfg, K)
    x = synth.config_vector(cfg, A.nrows, K)
    y = M.spmv(M.DeviceCsr(A, K, ctx=ctx), x, M.ORDER_FAST)
    ok, worst = bound_ok(A, x, y, _ref_real(A, x), K)
    print(f"cfg{cfg} K={K} rows={A.nrows} nnz={A.indptr[-1]} worst/bound={worst:.3g}")
    assert ok and worst <= MARGIN, worst


@pytest.mark.parametrize("K", [2, 4], ids=["cfg3_DD", "cfg3_QD"])
def test_fast_full_size_complex_within_bound(ctx, K):
    A = synth.config_matrix(3, K)
    xr, xi = synth.config_vector(3, A.nrows, K)
    yr, yi = M.spmv_complex(M.DeviceCsr(A, K, True, ctx=ctx), xr, xi, M.ORDER_FAST)
    rr, ri = _ref_complex(A, xr, xi)
    s = (O.abs_rowsum(A, A.planes[0], xr) + O.abs_rowsum(A, A.planes[K], xi) +
         O.abs_rowsum(A, A.planes[0], xi) + O.abs_rowsum(A, A.planes[K], xr))
    worst = 0.0
    for y, ref in ((yr, rr), (yi, ri)):
        ok, w = bound_ok(A, xr, y, ref, K, extra=s)
        assert ok, w
        worst = max(worst, w)
    print(f"cfg3 complex K={K} rows={A.nrows} worst/bound={worst:.3g}")
    assert worst <= MARGIN, worst
