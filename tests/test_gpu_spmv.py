"""GPU parity: the CUDA SpMV (through the C ABI) against the reference's golden
vectors and the pinned CPU oracle.  Deterministic orders must be bit-exact;
the fast order must satisfy |y - y_ref| <= 4 * rowlen * u * sum|a||x|
(u = 2^-104 / 2^-156 / 2^-208, BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle as O
import paper_2412_17510_b200 as M
import synth
from tests.util import U, bits_equal, bound_ok, csr, first_mismatch, golden, widen

pytestmark = pytest.mark.gpu

SMALL = {"cfg1": (1, 16, 0.0, 0.0), "cfg2": (2, 600, 32.0, 0.0), "cfg3": (3, 300, 32.0, 0.0),
         "cfg4": (4, 3000, 700.0, 1.8), "cfg5": (5, 6, 0.0, 0.0)}


@pytest.fixture(scope="module")
def ctx():
    c = M.Context(0)
    yield c
    c.close()


def _upload(ctx, A, K, cplx=False):
    return M.DeviceCsr(A, K, cplx, ctx=ctx)


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("order", [0, 1])
def test_worked_example(ctx, K, order):
    from tests.test_oracle import _example5x5

    A = widen(_example5x5(), K)
    x = np.zeros((5, K))
    x[:, 0] = np.arange(1, 6)
    y = M.spmv(_upload(ctx, A, K), x, order)
    assert bits_equal(y, golden("spmv_small")[f"ex5_K{K}_o{order}"])
    assert list(y[:, 0]) == [7.0, -14.0, 15.0, -22.0, 40.0]


@pytest.mark.parametrize("name", list(SMALL))
@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("order", [0, 1])
def test_small_configs_bit_exact(ctx, name, K, order):
    cfg, p1, p2, p3 = SMALL[name]
    A = synth.config_matrix(cfg, K, p1, p2, p3)
    g = golden("spmv_small")
    dA = _upload(ctx, A, K, cfg == 3)
    if cfg == 3:
        xr, xi = synth.config_vector(3, A.nrows, K)
        yr, yi = M.spmv_complex(dA, xr, xi, order)
        assert bits_equal(yr, g[f"{name}_K{K}_o{order}_re"]), first_mismatch(yr, g[f"{name}_K{K}_o{order}_re"])
        assert bits_equal(yi, g[f"{name}_K{K}_o{order}_im"]), first_mismatch(yi, g[f"{name}_K{K}_o{order}_im"])
    else:
        x = synth.config_vector(cfg, A.nrows, K)
        y = M.spmv(dA, x, order)
        assert bits_equal(y, g[f"{name}_K{K}_o{order}"]), first_mismatch(y, g[f"{name}_K{K}_o{order}"])


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("threshold", [4, 8, 33])
@pytest.mark.parametrize("order", [0, 1])
def test_long_row_store_bit_exact(K, threshold, order):
    """Force most rows through the long-row store (CTA per row, serial chains)."""
    c = M.Context(0)
    c.set_layout(long_threshold=threshold, sigma=64)
    for cfg in (2, 4):
        A = synth.config_matrix(cfg, K, *((500, 32.0, 0.0) if cfg == 2 else (2000, 900.0, 1.8)))
        x = synth.config_vector(cfg, A.nrows, K)
        y = M.spmv(M.DeviceCsr(A, K, ctx=c), x, order)
        ref = O.spmv(A, x, order)
        assert bits_equal(y, ref), first_mismatch(y, ref)
    A = synth.config_matrix(3, K, 200, 32.0)
    xr, xi = synth.config_vector(3, A.nrows, K)
    yr, yi = M.spmv_complex(M.DeviceCsr(A, K, True, ctx=c), xr, xi, order)
    rr, ri = O.spmv_complex(A, xr, xi, order)
    assert bits_equal(yr, rr) and bits_equal(yi, ri)
    c.close()


@pytest.mark.parametrize("K", [2, 3, 4])
def test_tub1000_and_qc324_fixtures(ctx, K):
    from tests.test_oracle import _tub1000

    g = golden("spmv_small")
    A = widen(_tub1000(), K)
    dA = _upload(ctx, A, K)
    for order in (0, 1):
        assert bits_equal(M.spmv(dA, g[f"make_vector_K{K}"], order), g[f"tub1000_K{K}_o{order}"])


@pytest.mark.parametrize("K", [2, 3, 4])
def test_edge_cases_empty_ragged_nonfinite(ctx, K):
    rng = np.random.default_rng(K)
    n = 97
    rows = []
    for i in range(n):
        L = int(rng.choice([0, 0, 1, 2, 3, 4, 5, 7, 31, 64, 300]))
        rows.append(sorted(rng.choice(n, size=min(L, n), replace=False).tolist()))
    A = csr(n, n, rows, K, seed=11)
    x = synth.vector(synth.VAL_NORMAL, n, K, seed=12)
    # non-finite and signed-zero inputs propagate exactly like the reference
    x[3] = [np.inf] + [0.0] * (K - 1)
    x[5] = [np.nan] + [0.0] * (K - 1)
    x[7] = [-0.0] * K
    x[9] = [0.0] + [-0.0] * (K - 1)
    A.planes[:, 2] = -0.0
    dA = _upload(ctx, A, K)
    for order in (0, 1):
        y = M.spmv(dA, x, order)
        ref = O.spmv(A, x, order)
        assert bits_equal(y, ref), first_mismatch(y, ref)


@pytest.mark.parametrize("K", [2, 3, 4])
def test_complex_ragged_rows_and_nonfinite(ctx, K):
    """Complex rows of every length 0..13 and a few longer ones (the DD kernel
    walks rounds of 5 elements, pairs in the LANE4 chains, with a partial last
    round), NaN / Inf / signed zeros in x: both exact orders bit for bit, FAST
    within the bound on the finite rows."""
    rng = np.random.default_rng(40 + K)
    n = 160
    lens = list(range(14)) * 8 + [17, 21, 26, 33, 64, 65, 66, 70] * 6
    rows = [sorted(rng.choice(n, size=L, replace=False).tolist()) for L in lens[:n]]
    A = csr(n, n, rows, K, seed=21, is_complex=True)
    xr = synth.vector(synth.VAL_NORMAL, n, K, seed=22)
    xi = synth.vector(synth.VAL_NORMAL, n, K, seed=23)
    dA = _upload(ctx, A, K, cplx=True)
    yr, yi = M.spmv_complex(dA, xr, xi, M.ORDER_FAST)
    rr, ri = O.spmv_complex(A, xr, xi, 0)
    s = (O.abs_rowsum(A, A.planes[0], xr) + O.abs_rowsum(A, A.planes[K], xi) +
         O.abs_rowsum(A, A.planes[0], xi) + O.abs_rowsum(A, A.planes[K], xr))
    for y, ref in ((yr, rr), (yi, ri)):
        ok, worst = bound_ok(A, xr, y, ref, K, extra=s)
        assert ok and worst <= 0.25, worst
    xr[3] = [np.inf] + [0.0] * (K - 1)
    xi[5] = [np.nan] + [0.0] * (K - 1)
    xr[7] = [-0.0] * K
    xi[9] = [0.0] + [-0.0] * (K - 1)
    for order in (0, 1):
        yr, yi = M.spmv_complex(dA, xr, xi, order)
        rr, ri = O.spmv_complex(A, xr, xi, order)
        assert bits_equal(yr, rr), first_mismatch(yr, rr)
        assert bits_equal(yi, ri), first_mismatch(yi, ri)


def test_empty_and_zero_nnz_matrices(ctx):
    A = csr(0, 0, [], 2)
    y = M.spmv(_upload(ctx, A, 2), np.zeros((0, 2)), 1)
    assert y.shape == (0, 2)
    A = csr(5, 3, [[], [], [], [], []], 4)
    y = M.spmv(_upload(ctx, A, 4), np.ones((3, 4)), 1)
    assert bits_equal(y, np.zeros((5, 4)))


def test_dimension_mismatch_message(ctx):
    A = csr(4, 4, [[0], [1], [2], [3]], 2)
    dA = _upload(ctx, A, 2)
    with pytest.raises(ValueError, match="spmv: vector length 3 does not match matrix dimension 4"):
        M.spmv(dA, np.zeros((3, 2)), 1)


def test_out_of_range_column_rejected(ctx):
    A = csr(3, 3, [[0], [5], [2]], 2)
    with pytest.raises(M.MpsgError) as e:
        _upload(ctx, A, 2)
    assert e.value.code == M.E_RANGE


@pytest.mark.parametrize("name,K", [("cfg1", 2), ("cfg2", 3), ("cfg2", 4), ("cfg4", 2), ("cfg5", 2),
                                    ("cfg5", 4)])
@pytest.mark.parametrize("order", [0, 1])
def test_full_size_checksums(ctx, name, K, order):
    """BASELINE.json full sizes: FNV-1a checksum equals the reference's."""
    cfg = int(name[3])
    g = golden("spmv_full")
    A = synth.config_matrix(cfg, K)
    x = synth.config_vector(cfg, A.nrows, K)
    y = M.spmv(_upload(ctx, A, K), x, order)
    assert M.checksum(y) == int(g[f"{name}_K{K}_o{order}"])


@pytest.mark.parametrize("K", [2, 4])
@pytest.mark.parametrize("order", [0, 1])
def test_full_size_complex_checksum(ctx, K, order):
    g = golden("spmv_full")
    A = synth.config_matrix(3, K)
    xr, xi = synth.config_vector(3, A.nrows, K)
    yr, yi = M.spmv_complex(_upload(ctx, A, K, True), xr, xi, order)
    assert M.checksum_complex(yr, yi) == int(g[f"cfg3_K{K}_o{order}"])


@pytest.mark.parametrize("K", [2, 3, 4])
def test_fast_order_within_bound(ctx, K):
    c = M.Context(0)
    c.set_layout(long_threshold=16, sigma=256, fast_chunk=64)
    A = synth.config_matrix(4, K, 3000, 2000.0, 1.8)
    x = synth.config_vector(4, A.nrows, K)
    y = M.spmv(M.DeviceCsr(A, K, ctx=c), x, M.ORDER_FAST)
    ref = O.spmv(A, x, 1)
    ok, worst = bound_ok(A, x, y, ref, K)
    assert ok, worst
    c.close()


@pytest.mark.parametrize("K", [2, 4])
def test_fast_order_complex_within_bound(K):
    c = M.Context(0)
    c.set_layout(long_threshold=8, sigma=256, fast_chunk=32)
    A = synth.config_matrix(3, K, 400, 40.0)
    xr, xi = synth.config_vector(3, A.nrows, K)
    yr, yi = M.spmv_complex(M.DeviceCsr(A, K, True, ctx=c), xr, xi, M.ORDER_FAST)
    rr, ri = O.spmv_complex(A, xr, xi, 1)
    s = (O.abs_rowsum(A, A.planes[0], xr) + O.abs_rowsum(A, A.planes[K], xi) +
         O.abs_rowsum(A, A.planes[0], xi) + O.abs_rowsum(A, A.planes[K], xr))
    assert bound_ok(A, xr, yr, rr, K, extra=s)[0]
    assert bound_ok(A, xr, yi, ri, K, extra=s)[0]
    c.close()


def test_fast_full_cfg4_within_bound(ctx):
    A = synth.config_matrix(4, 2)
    x = synth.config_vector(4, A.nrows, 2)
    dA = _upload(ctx, A, 2)
    assert dA.stats().nlong > 0
    y = M.spmv(dA, x, M.ORDER_FAST)
    yl = M.spmv(dA, x, M.ORDER_LANE4)
    assert M.checksum(yl) == int(golden("spmv_full")["cfg4_K2_o1"])
    # check the bound on the long rows (short rows are computed in reference order)
    st = np.diff(A.indptr)
    rows = np.nonzero(st > 256)[0]
    sub = _row_subset(A, rows)
    ok, worst = bound_ok(sub, x, y[rows], yl[rows], 2)
    assert ok, worst


def _row_subset(A, rows):
    from types import SimpleNamespace

    lens = np.diff(A.indptr)[rows]
    indptr = np.concatenate([[0], np.cumsum(lens)])
    idx = np.concatenate([np.arange(A.indptr[r], A.indptr[r + 1]) for r in rows])
    return SimpleNamespace(nrows=len(rows), ncols=A.ncols, indptr=indptr, indices=A.indices[idx],
                           planes=A.planes[:, idx])


def test_device_pointer_entry_and_stream():
    """mpsg_spmv_dev on caller-owned device memory and a caller stream (torch plumbing)."""
    import torch

    c = M.Context(0)
    A = synth.config_matrix(2, 4, 2000)
    x = synth.config_vector(2, A.nrows, 4)
    dA = M.DeviceCsr(A, 4, ctx=c)
    dx = torch.from_numpy(x).cuda()
    dy = torch.empty_like(dx)
    s = torch.cuda.Stream()
    M.spmv_dev(dA, dx.data_ptr(), dy.data_ptr(), M.ORDER_LANE4, s.cuda_stream)
    s.synchronize()
    assert bits_equal(dy.cpu().numpy(), O.spmv(A, x, 1))
    c.close()


@pytest.mark.parametrize("K", [2, 4])
@pytest.mark.parametrize("order", [0, 1, 2])
def test_host_call_overlapped_parts(K, order):
    """Host-pointer calls copy y back part by part while later parts compute
    (many sort windows -> 8 parts); results identical to the oracle /
    the device-pointer path, with and without long rows, real and complex."""
    import torch

    c = M.Context(0)
    c.set_layout(long_threshold=40, sigma=64)
    for cfg, args in ((2, (2000, 32.0, 0.0)), (4, (3000, 700.0, 1.8))):
        A = synth.config_matrix(cfg, K, *args)
        x = synth.config_vector(cfg, A.nrows, K)
        dA = M.DeviceCsr(A, K, ctx=c)
        y = M.spmv(dA, x, order)
        dx = torch.from_numpy(x).cuda()
        dy = torch.empty_like(dx[: A.nrows])
        M.spmv_dev(dA, dx.data_ptr(), dy.data_ptr(), order, None)
        c.synchronize()
        assert bits_equal(y, dy.cpu().numpy())
        if order < 2:
            assert bits_equal(y, O.spmv(A, x, order))
    A = synth.config_matrix(3, K, 1500, 16.0)
    xr, xi = synth.config_vector(3, A.nrows, K)
    yr, yi = M.spmv_complex(M.DeviceCsr(A, K, True, ctx=c), xr, xi, order)
    if order < 2:
        rr, ri = O.spmv_complex(A, xr, xi, order)
        assert bits_equal(yr, rr) and bits_equal(yi, ri)
    c.close()


@pytest.mark.parametrize("order", [0, 1, 2])
def test_unaligned_device_x_takes_the_narrow_gather(order):
    """QD x gathers use 256-bit loads only when x is 32-byte aligned; an x
    that starts 16 bytes into an allocation (the ABI's minimum alignment for
    DD / QD device vectors) must give the same result, and an 8-byte offset is
    refused (MPSG_E_ARG) instead of faulting."""
    import torch

    c = M.Context(0)
    K = 4
    A = synth.config_matrix(2, K, 3000)
    x = synth.config_vector(2, A.nrows, K)
    dA = M.DeviceCsr(A, K, ctx=c)
    flat = torch.zeros(A.nrows * K + 2, dtype=torch.float64, device="cuda")
    flat[2:] = torch.from_numpy(x.reshape(-1)).cuda()
    assert (flat.data_ptr() + 16) % 32 != 0
    dy = torch.empty((A.nrows, K), dtype=torch.float64, device="cuda")
    M.spmv_dev(dA, flat.data_ptr() + 16, dy.data_ptr(), order, None)
    c.synchronize()
    aligned = M.spmv(dA, x, order)
    assert bits_equal(dy.cpu().numpy(), aligned)
    if order != 2:
        assert bits_equal(aligned, O.spmv(A, x, order))
    with pytest.raises(M.MpsgError) as ei:
        M.spmv_dev(dA, flat.data_ptr() + 8, dy.data_ptr(), order, None)
    assert ei.value.code == 6 and "aligned" in str(ei.value)
    c.close()
