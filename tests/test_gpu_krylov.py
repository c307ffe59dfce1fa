"""GPU parity for the device-resident Krylov solvers (solve(), krylov.hpp:
238-606: CG, BiCG, CGS, BiCGSTAB, GPBiCG) through the C ABI mpsg_solve.

Two tiers, as for CG:
  * exact dots (SolverConfig.exact_dots: one device thread per dot, the
    reference's sequential order) with an exact SpMV order -> the solve is the
    reference's, bit for bit: iterate, residual history, iteration count,
    status, detail text, rhs norm and final true residual, on every case of
    the reference golden (tests/golden/krylov_small.npz, generated from the
    reference's own solve()), including every breakdown exit, the half-step
    exits, x0 starts and MaxIterations;
  * tree dots (default, throughput) -> same status and detail, iteration count
    within +-1 (the cases converge in 20-40 iterations, so the north star's
    1% is below one iteration), final true residual at the reference's level.
"""
import numpy as np
import pytest

import oracle as O
import paper_2412_17510_b200 as M
from tests.util import bits_equal, golden, krylov_cases, krylov_system

pytestmark = pytest.mark.gpu

_KCASES = krylov_cases()


@pytest.fixture(scope="module")
def ctx():
    c = M.Context(0)
    yield c
    c.close()


def _run(ctx, A, b, method, exact=True, order=M.ORDER_LANE4, use_graph=True, check_every=32, **kw):
    K = b.shape[1]
    dA = M.DeviceCsr(A, K, ctx=ctx, transpose=(method == "bicg"))
    op = M.CsrOperator(dA, threads=kw.pop("threads", 1), lanes_enabled=order != M.ORDER_SCALAR,
                       fast=order == M.ORDER_FAST)
    cfg = M.SolverConfig(method=M.parse_method(method), exact_dots=exact, use_graph=use_graph,
                         check_every=check_every, **kw)
    return M.solve(op, b, cfg)


@pytest.mark.parametrize("case", _KCASES, ids=[c[0] for c in _KCASES])
def test_solve_exact_dots_bit_equal_reference(ctx, case):
    name, A, b, m, kw = case
    g = golden("krylov_small")
    res = _run(ctx, A, b, m, exact=True, **dict(kw))
    rep = res.report
    meta = g[f"{name}_meta"]
    assert (rep.iterations, int(rep.status)) == (int(meta[0]), int(meta[1])), (rep.iterations, rep.status, meta)
    assert rep.detail == str(g[f"{name}_detail"])
    assert len(rep.residual_history) == rep.iterations + 1
    assert bits_equal(np.array(rep.residual_history), g[f"{name}_history"])
    assert bits_equal(res.x, g[f"{name}_x"])
    assert bits_equal(np.array([rep.rhs_norm, rep.final_true_residual]), meta[2:])
    assert rep.converged == (int(meta[1]) == 0)
    assert rep.final_recurrence_residual == rep.residual_history[-1] or np.isnan(rep.final_recurrence_residual)


@pytest.mark.parametrize("order", [M.ORDER_LANE4, M.ORDER_FAST], ids=["lane4", "fast"])
@pytest.mark.parametrize("case", _KCASES, ids=[c[0] for c in _KCASES])
def test_solve_tree_dots_tracks_reference(ctx, case, order):
    """order FAST also runs the fused product-accumulates (TD/QD)."""
    name, A, b, m, kw = case
    g = golden("krylov_small")
    res = _run(ctx, A, b, m, exact=False, order=order, **dict(kw))
    rep = res.report
    meta = g[f"{name}_meta"]
    ref_iters, ref_status = int(meta[0]), int(meta[1])
    if ref_status == 2 and ref_iters > 2:
        # a breakdown reached only after many iterations of round-off (a
        # near-singular recurrence) depends on the dot rounding order; it is
        # pinned by the exact-dots tier above
        pytest.skip("round-off-driven breakdown: exact-dots tier only")
    assert int(rep.status) == ref_status, (rep.status, rep.detail, meta, str(g[f"{name}_detail"]))
    assert rep.detail == str(g[f"{name}_detail"])
    assert abs(rep.iterations - ref_iters) <= 1, (rep.iterations, ref_iters)
    assert len(rep.residual_history) == rep.iterations + 1
    ref_h = g[f"{name}_history"]
    assert rep.residual_history[0] == ref_h[0] and rep.rhs_norm == meta[2]
    if ref_status == 0:
        # converged: the true residual is at the reference's level
        assert rep.final_true_residual <= max(10 * meta[3], 1e-13 * meta[2] + 1e-99)


@pytest.mark.parametrize("m", O.METHODS)
def test_solve_graph_and_batches_do_not_change_bits(ctx, m):
    A, b = krylov_system(60, 3, seed=3, symmetric=m == "cg")
    r1 = _run(ctx, A, b, m, exact=True, use_graph=True, check_every=32)
    r2 = _run(ctx, A, b, m, exact=True, use_graph=False, check_every=5)
    r3 = _run(ctx, A, b, m, exact=False, use_graph=True, check_every=3)
    r4 = _run(ctx, A, b, m, exact=False, use_graph=False, check_every=64)
    assert bits_equal(r1.x, r2.x) and r1.report.residual_history == r2.report.residual_history
    assert bits_equal(r3.x, r4.x) and r3.report.residual_history == r4.report.residual_history


@pytest.mark.parametrize("m", O.METHODS)
@pytest.mark.parametrize("order", [M.ORDER_SCALAR, M.ORDER_LANE4])
def test_solve_exact_matches_oracle_larger(ctx, m, order):
    """A multi-block system (n = 3000, rows of 1-40 nonzeros so both SpMV orders
    differ) against the oracle's C restatement of solve()."""
    A, b = krylov_system(3000, 2, seed=11, symmetric=m == "cg", density=0.004)
    kw = dict(rel_tol=1e-25, max_iters=40)
    res = _run(ctx, A, b, m, exact=True, order=order, threads=3 if m == "bicg" else 1, **kw)
    ref = O.solve(A, b, m, order=order, threads=3 if m == "bicg" else 1, **kw)
    assert (res.report.iterations, int(res.report.status)) == (ref["iterations"], ref["status"])
    assert bits_equal(np.array(res.report.residual_history), ref["history"])
    assert bits_equal(res.x, ref["x"])
    assert res.report.final_true_residual == ref["final_true_residual"]


@pytest.mark.parametrize("m", O.METHODS)
def test_solve_fast_order_converges(ctx, m):
    A, b = krylov_system(2000, 4, seed=5, symmetric=m == "cg", density=0.01)
    ref = O.solve(A, b, m, rel_tol=1e-50, max_iters=200)
    res = _run(ctx, A, b, m, exact=False, order=M.ORDER_FAST, rel_tol=1e-50, max_iters=200)
    assert res.report.converged and ref["status"] == 0
    assert abs(res.report.iterations - ref["iterations"]) <= max(1, ref["iterations"] // 100)
    assert res.report.final_true_residual < 1e-45


def test_solve_errors(ctx):
    A, b = krylov_cases()[0][1:3]
    dA = M.DeviceCsr(A, b.shape[1], ctx=ctx)
    op = M.CsrOperator(dA)
    with pytest.raises(ValueError, match="tolerances must be positive"):
        M.solve(op, b, M.SolverConfig(rel_tol=0.0))
    with pytest.raises(ValueError, match="max_iters"):
        M.solve(op, b, M.SolverConfig(max_iters=0))
    with pytest.raises(ValueError, match="rhs length"):
        M.solve(op, b[:-1], M.SolverConfig())
    with pytest.raises(M.MpsgError, match="MPSG_CSR_TRANSPOSE"):
        M.solve_bicg(op, b)
    # the default method is BiCGSTAB (krylov.hpp:59)
    assert M.SolverConfig().method == M.KrylovMethod.BiCGSTAB
    assert str(M.KrylovMethod.GPBiCG) == "gpbicg" and M.parse_method("cgs") == M.KrylovMethod.CGS


# ---- Mixed mode: solve() over CsrOperator<double> with K-component vectors ------
from tests.util import krylov_mixed_cases  # noqa: E402

_MCASES = krylov_mixed_cases()


@pytest.mark.parametrize("case", _MCASES, ids=[c[0] for c in _MCASES])
def test_mixed_solve_exact_dots_bit_equal_reference(ctx, case):
    name, Am, b, m, kw = case
    g = golden("krylov_mixed")
    K = b.shape[1]
    dA = M.DeviceCsr(Am, K, ctx=ctx, mixed=True, transpose=(m == "bicg"))
    op = M.CsrOperator(dA, threads=kw.get("threads", 1))
    res = M.solve(op, b, M.SolverConfig(method=M.parse_method(m), exact_dots=True))
    meta = g[f"{name}_meta"]
    assert (res.report.iterations, int(res.report.status)) == (int(meta[0]), int(meta[1]))
    assert bits_equal(np.array(res.report.residual_history), g[f"{name}_history"])
    assert bits_equal(res.x, g[f"{name}_x"])
    assert res.report.final_true_residual == meta[3] and res.report.detail == str(g[f"{name}_detail"])


# ---- edge cases: empty and 1x1 systems, a single iteration, x0 = exact ------------
@pytest.mark.parametrize("m", O.METHODS)
@pytest.mark.parametrize("exact", [True, False])
def test_solve_edge_cases_match_oracle(ctx, m, exact):
    from tests.util import csr, dense_system

    cases = []
    cases.append(("one", *dense_system([[3.0]], [1.5]), {}))
    cases.append(("one_iter", *krylov_system(40, 2, seed=4, symmetric=m == "cg"), {"max_iters": 1}))
    D, bd = dense_system(np.diag([2.0, 4.0, 8.0]), [2.0, 4.0, 8.0])
    cases.append(("x0_exact", D, bd, {"x0": [1.0, 1.0, 1.0]}))
    cases.append(("zero_rhs", D, np.zeros_like(bd), {}))
    for name, A, b, kw in cases:
        r = _run(ctx, A, b, m, exact=exact, **dict(kw))
        ref = O.solve(A, b, m, **kw)
        assert (r.report.iterations, int(r.report.status)) == (ref["iterations"], ref["status"]), name
        assert r.report.detail == ref["detail"], name
        if exact:
            assert bits_equal(np.array(r.report.residual_history), ref["history"]), name
            assert bits_equal(r.x, ref["x"]), name


def test_solve_empty_system(ctx):
    from tests.util import csr

    A = csr(0, 0, [], 2)
    b = np.zeros((0, 2))
    for m in O.METHODS:
        r = _run(ctx, A, b, m, exact=False)
        assert r.report.converged and r.report.iterations == 0 and r.x.shape == (0, 2)
