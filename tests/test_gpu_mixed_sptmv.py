"""GPU parity for the §8(f) rows beside the Pure SpMV: Mixed mode (binary64
matrix x multi-component vector, kernels.hpp:55-58, 123-142) and the
transposed products sptmv / sptmv_complex (+ adjoint) (kernels.hpp:368-441).
Exact orders bit-for-bit against the oracle (itself pinned to the reference in
tests/test_oracle.py and by tests/golden/mixed_sptmv.npz); FAST within the
componentwise bound."""
import numpy as np
import pytest

import oracle as O
import paper_2412_17510_b200 as M
import synth
from tests.util import bits_equal, bound_ok, first_mismatch, golden, mixed_of, transpose

pytestmark = pytest.mark.gpu

CASES = {"cfg2": (2, 600, 32.0, 0.0), "cfg4": (4, 3000, 700.0, 1.8), "cfg5": (5, 6, 0.0, 0.0)}


@pytest.fixture(scope="module")
def ctx():
    c = M.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("order", [0, 1])
def test_mixed_spmv_bit_exact(ctx, name, K, order):
    A = mixed_of(synth.config_matrix(*((CASES[name][0], K) + CASES[name][1:])))
    x = synth.config_vector(CASES[name][0], A.nrows, K)
    y = M.spmv(M.DeviceCsr(A, K, ctx=ctx, mixed=True), x, order)
    ref = O.spmv(A, x, order, mixed=True)
    assert bits_equal(y, ref), first_mismatch(y, ref)


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("order", [0, 1])
def test_mixed_long_rows_and_complex(K, order):
    c = M.Context(0)
    c.set_layout(long_threshold=16, sigma=128)
    A = mixed_of(synth.config_matrix(4, K, 2000, 900.0, 1.8))
    x = synth.config_vector(4, A.nrows, K)
    y = M.spmv(M.DeviceCsr(A, K, ctx=c, mixed=True), x, order)
    assert bits_equal(y, O.spmv(A, x, order, mixed=True))
    C = mixed_of(synth.config_matrix(3, K, 300, 24.0), cplx=True)
    xr, xi = synth.config_vector(3, C.nrows, K)
    yr, yi = M.spmv_complex(M.DeviceCsr(C, K, True, ctx=c, mixed=True), xr, xi, order)
    rr, ri = O.spmv_complex(C, xr, xi, order, mixed=True)
    assert bits_equal(yr, rr) and bits_equal(yi, ri)
    c.close()


@pytest.mark.parametrize("K", [2, 3, 4])
def test_mixed_fast_within_bound(K):
    c = M.Context(0)
    c.set_layout(long_threshold=16, sigma=256, fast_chunk=64)
    A = mixed_of(synth.config_matrix(4, K, 3000, 2000.0, 1.8))
    x = synth.config_vector(4, A.nrows, K)
    y = M.spmv(M.DeviceCsr(A, K, ctx=c, mixed=True), x, M.ORDER_FAST)
    ok, worst = bound_ok(A, x, y, O.spmv(A, x, 1, mixed=True), K)
    assert ok, worst
    c.close()


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("mixed", [False, True])
def test_sptmv_bit_exact(ctx, name, K, order, mixed):
    A = synth.config_matrix(*((CASES[name][0], K) + CASES[name][1:]))
    if mixed:
        A = mixed_of(A)
    v = synth.config_vector(CASES[name][0], A.nrows, K)
    y = M.sptmv(M.DeviceCsr(A, K, ctx=ctx, mixed=mixed, transpose=True), v, order)
    ref = O.sptmv(A, v, threads=1, mixed=mixed)  # the reference at one thread, lanes on or off
    assert bits_equal(y, ref), first_mismatch(y, ref)


@pytest.mark.parametrize("K", [2, 4])
@pytest.mark.parametrize("conjugate", [False, True])
@pytest.mark.parametrize("mixed", [False, True])
def test_sptmv_complex_bit_exact(ctx, K, conjugate, mixed):
    A = synth.config_matrix(3, K, 300, 24.0)
    if mixed:
        A = mixed_of(A, cplx=True)
    vr, vi = synth.config_vector(3, A.nrows, K)
    dA = M.DeviceCsr(A, K, True, ctx=ctx, mixed=mixed, transpose=True)
    for order in (0, 1):
        yr, yi = M.sptmv_complex(dA, vr, vi, order, conjugate=conjugate)
        rr, ri = O.sptmv_complex(A, vr, vi, 1, conjugate, mixed)
        assert bits_equal(yr, rr) and bits_equal(yi, ri)


def test_sptmv_long_columns_and_fast_bound():
    """A dense column makes a long row of A^T: exact order through the long
    store, FAST within the bound."""
    c = M.Context(0)
    c.set_layout(long_threshold=64)
    K = 4
    A = synth.config_matrix(2, K, 3000, 8.0)
    # add column 7 to every row (keeps columns sorted/unique per row)
    rows = [sorted(set(A.indices[A.indptr[i]:A.indptr[i + 1]].tolist()) | {7}) for i in range(A.nrows)]
    from tests.util import csr

    B = csr(A.nrows, A.ncols, rows, K, seed=5)
    v = synth.vector(synth.VAL_NORMAL, B.nrows, K, seed=9)
    dB = M.DeviceCsr(B, K, ctx=c, transpose=True)
    assert dB.stats().has_transpose
    for order in (0, 1):
        assert bits_equal(M.sptmv(dB, v, order), O.sptmv(B, v))
    yf = M.sptmv(dB, v, M.ORDER_FAST)
    T = transpose(B)
    ok, worst = bound_ok(T, v, yf, O.sptmv(B, v), K)
    assert ok, worst
    c.close()


def test_sptmv_requires_transpose_upload(ctx):
    A = synth.config_matrix(2, 2, 200)
    v = synth.config_vector(2, A.nrows, 2)
    with pytest.raises(M.MpsgError, match="TRANSPOSE"):
        M.sptmv(M.DeviceCsr(A, 2, ctx=ctx), v)


def test_sptmv_dimension_message(ctx):
    A = synth.config_matrix(2, 2, 200)
    dA = M.DeviceCsr(A, 2, ctx=ctx, transpose=True)
    with pytest.raises(ValueError, match=r"sptmv: vector length 5 does not match matrix dimension 200"):
        M.sptmv(dA, np.zeros((5, 2)))


def test_operator_apply_transposed(ctx):
    A = synth.config_matrix(5, 2, 6)
    v = synth.config_vector(5, A.nrows, 2)
    op = M.CsrOperator(M.DeviceCsr(A, 2, ctx=ctx, transpose=True))
    assert bits_equal(op.apply_transposed(v), O.sptmv(A, v))


@pytest.mark.parametrize("key", ["mixed_cfg2_K4_o1", "mixed_cfg4_K2_o0", "sptmv_cfg2_K3", "sptmv_mixed_cfg4_K2",
                                 "csptmv_K4_conj"])
def test_against_reference_goldens(ctx, key):
    g = golden("mixed_sptmv")
    if key.startswith("mixed_"):
        _, name, k, o = key.split("_")
        K, order = int(k[1]), int(o[1])
        cfg = CASES[name]
        A = mixed_of(synth.config_matrix(*((cfg[0], K) + cfg[1:])))
        x = synth.config_vector(cfg[0], A.nrows, K)
        y = M.spmv(M.DeviceCsr(A, K, ctx=ctx, mixed=True), x, order)
        assert bits_equal(y, g[key])
    elif key.startswith("sptmv"):
        parts = key.split("_")
        mixed = parts[1] == "mixed"
        name, K = parts[-2], int(parts[-1][1])
        cfg = CASES[name]
        A = synth.config_matrix(*((cfg[0], K) + cfg[1:]))
        if mixed:
            A = mixed_of(A)
        v = synth.config_vector(cfg[0], A.nrows, K)
        y = M.sptmv(M.DeviceCsr(A, K, ctx=ctx, mixed=mixed, transpose=True), v, 1)
        assert bits_equal(y, g[key])
    else:
        K = 4
        A = synth.config_matrix(3, K, 300, 24.0)
        vr, vi = synth.config_vector(3, A.nrows, K)
        yr, yi = M.sptmv_complex(M.DeviceCsr(A, K, True, ctx=ctx, transpose=True), vr, vi, 1, conjugate=True)
        assert bits_equal(yr, g[key + "_re"]) and bits_equal(yi, g[key + "_im"])


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("threads", [2, 3, 5, 16])
@pytest.mark.parametrize("mixed", [False, True])
def test_sptmv_thread_count_merge_bit_exact(K, threads, mixed):
    """The reference sptmv at T threads: per-thread accumulators merged in thread
    order (oracle restatement pinned to the reference for T = 1, 2, 5)."""
    c = M.Context(0)
    c.set_layout(long_threshold=64)
    A = synth.config_matrix(4, K, 3000, 800.0, 1.8)
    rows = [sorted(set(A.indices[A.indptr[i]:A.indptr[i + 1]].tolist()) | {3}) for i in range(A.nrows)]
    from tests.util import csr

    B = csr(A.nrows, A.ncols, rows, K, seed=2)  # dense column 3: a long row of B^T
    if mixed:
        B = mixed_of(B)
    v = synth.vector(synth.VAL_NORMAL, B.nrows, K, seed=4)
    dB = M.DeviceCsr(B, K, ctx=c, mixed=mixed, transpose=True)
    for order in (0, 1):
        y = M.sptmv(dB, v, M.KernelMode(threads=threads, lanes_enabled=order == 1))
        ref = O.sptmv(B, v, threads=threads, mixed=mixed)
        assert bits_equal(y, ref), first_mismatch(y, ref)
    C = synth.config_matrix(3, K, 400, 24.0)
    vr, vi = synth.config_vector(3, C.nrows, K)
    dC = M.DeviceCsr(C, K, True, ctx=c, transpose=True)
    for conj in (False, True):
        yr, yi = M.sptmv_complex(dC, vr, vi, M.KernelMode(threads=threads), conjugate=conj)
        rr, ri = O.sptmv_complex(C, vr, vi, threads, conj)
        assert bits_equal(yr, rr) and bits_equal(yi, ri)
    c.close()
