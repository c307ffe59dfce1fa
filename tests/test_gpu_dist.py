"""Row-sharded path (mpsg_comm / mpsg_dcsr) on one B200.

Only one GPU is available to the tests, so the NCCL layer runs as a one-rank
group: the shard is the whole matrix, the halo plan is empty, and the results
must equal the single-GPU path -- bit for bit for SpMV, iteration for
iteration for CG.  The multi-rank host logic (partition, plan, exchange) is
pinned on CPU by tests/test_dist_cpu.py.
"""
import numpy as np
import pytest

import oracle as O
import paper_2412_17510_b200 as M
import synth
from tests.util import bits_equal, csr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = M.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("cfg,K,p1,p2,p3", [(4, 2, 20000, 5000.0, 1.8), (5, 4, 24, 0.0, 0.0), (2, 3, 5000, 32.0, 0.0)])
@pytest.mark.parametrize("order", [0, 1])
def test_one_rank_dspmv_equals_spmv(ctx, cfg, K, p1, p2, p3, order):
    A = synth.config_matrix(cfg, K, p1, p2, p3)
    x = synth.config_vector(cfg, A.nrows, K)
    comm = M.Comm(ctx, 1, 0)
    dA = M.DistCsr.from_global(comm, A, K)
    bounds, halo = dA.info()
    assert bounds.tolist() == [0, A.nrows] and halo == 0
    y = M.dspmv(dA, x, order)
    assert bits_equal(y, O.spmv(A, x, order))
    dA.close()
    comm.close()


def test_one_rank_dspmv_complex_dev(ctx):
    import torch

    K = 4
    A = synth.config_matrix(3, K, 2000, 16.0)
    xr, xi = synth.config_vector(3, A.nrows, K)
    comm = M.Comm(ctx, 1, 0)
    dA = M.DistCsr.from_global(comm, A, K, is_complex=True)
    dxr, dxi = torch.from_numpy(xr).cuda(), torch.from_numpy(xi).cuda()
    dyr, dyi = torch.empty_like(dxr), torch.empty_like(dxi)
    M.dspmv_complex_dev(dA, dxr.data_ptr(), dxi.data_ptr(), dyr.data_ptr(), dyi.data_ptr(), M.ORDER_LANE4)
    ctx.synchronize()
    rr, ri = O.spmv_complex(A, xr, xi, 1)
    assert bits_equal(dyr.cpu().numpy(), rr) and bits_equal(dyi.cpu().numpy(), ri)


@pytest.mark.parametrize("variant", [0, 2], ids=["classic", "one_reduction"])
@pytest.mark.parametrize("K", [2, 4])
def test_one_rank_dcg_tracks_single_gpu_cg(ctx, K, variant):
    """NCCL one-rank group, iterations captured in CUDA graphs (the allgathers
    of the dot partials are inside the graph); variant 2 forces the
    one-reduction form through the sharded driver (prologue-folded scalars)."""
    A = synth.config_matrix(5, K, 20)
    xt = synth.config_vector(5, A.nrows, K)
    b = O.spmv(A, xt, 1)
    cfg = M.SolverConfig(rel_tol=1e-25, max_iters=300)
    single = M.solve_cg(M.CsrOperator(M.DeviceCsr(A, K, ctx=ctx)), b, cfg)
    comm = M.Comm(ctx, 1, 0)
    dA = M.DistCsr.from_global(comm, A, K)
    dist = M.dsolve_cg(dA, b, M.SolverConfig(rel_tol=1e-25, max_iters=300, cg_variant=variant))
    assert dist.report.status == single.report.status
    assert abs(dist.report.iterations - single.report.iterations) <= 1
    h1, h2 = np.array(single.report.residual_history), np.array(dist.report.residual_history)
    n = min(len(h1), len(h2)) - 5
    assert np.allclose(h1[:n], h2[:n], rtol=1e-10 if variant == 0 else 1e-3, atol=0)
    assert dist.report.final_true_residual <= 10 * single.report.final_true_residual + 1e-30


def test_one_rank_dcg_with_initial_guess_and_graph_off(ctx):
    K = 2
    A = synth.config_matrix(5, K, 12)
    xt = synth.config_vector(5, A.nrows, K)
    b = O.spmv(A, xt, 1)
    x0 = list(np.linspace(-1, 1, A.nrows))
    comm = M.Comm(ctx, 1, 0)
    dA = M.DistCsr.from_global(comm, A, K)
    r1 = M.dsolve_cg(dA, b, M.SolverConfig(rel_tol=1e-20, max_iters=200, x0=x0, use_graph=False))
    r2 = M.solve_cg(M.CsrOperator(M.DeviceCsr(A, K, ctx=ctx)), b, M.SolverConfig(rel_tol=1e-20, max_iters=200, x0=x0))
    assert r1.report.converged and r2.report.converged
    assert abs(r1.report.iterations - r2.report.iterations) <= 1
    assert np.allclose(r1.x[:, 0], xt[:, 0], atol=1e-12)


# ---- several ranks on one GPU: the single-process group backend ------------------
def _run_ranks(P, fn):
    """fn(rank, comm, ctx) on P host threads, one context and comm per rank."""
    import threading

    ctxs = [M.Context(0) for _ in range(P)]
    comms = M.Comm.local_group(ctxs)
    out, errs = [None] * P, []

    def body(r):
        try:
            out[r] = fn(r, comms[r], ctxs[r])
        except Exception as e:  # noqa: BLE001
            errs.append((r, repr(e)))

    ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    for c in comms:
        c.close()
    for c in ctxs:
        c.close()
    return out


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("cfg,K,p1,p2,p3", [(4, 2, 20000, 5000.0, 1.8), (5, 4, 24, 0.0, 0.0), (2, 3, 5000, 32.0, 0.0)])
def test_sharded_spmv_several_ranks_bit_exact(P, cfg, K, p1, p2, p3):
    A = synth.config_matrix(cfg, K, p1, p2, p3)
    x = synth.config_vector(cfg, A.nrows, K)
    bounds = M.partition_rows(A.indptr, A.nrows, P)

    def rank_fn(r, comm, ctx):
        dA = M.DistCsr.from_global(comm, A, K, bounds=bounds)
        b, e = dA.row_begin, dA.row_end
        res = {o: M.dspmv(dA, x[b:e], o) for o in (0, 1, 2)}
        res["interior"] = dA.interior_rows()
        dA.close()
        return res

    parts = _run_ranks(P, rank_fn)
    if cfg == 5:  # stencil: most rows are interior, computed while the halo moves
        assert all(p["interior"] > 0 for p in parts)
    for o in (0, 1):
        y = np.concatenate([p[o] for p in parts])
        assert bits_equal(y, O.spmv(A, x, o)), (P, o)
    # FAST: same kernels per shard, long rows reordered -> equal to the single-GPU FAST result
    yf = np.concatenate([p[2] for p in parts])
    assert bits_equal(yf, M.spmv(M.DeviceCsr(A, K), x, 2))


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_complex_several_ranks(P):
    import torch

    K = 2
    A = synth.config_matrix(3, K, 3000, 16.0)
    xr, xi = synth.config_vector(3, A.nrows, K)
    bounds = M.partition_rows(A.indptr, A.nrows, P)

    def rank_fn(r, comm, ctx):
        dA = M.DistCsr.from_global(comm, A, K, is_complex=True, bounds=bounds)
        b, e = dA.row_begin, dA.row_end
        with torch.cuda.device(0):
            dxr, dxi = torch.from_numpy(xr[b:e].copy()).cuda(), torch.from_numpy(xi[b:e].copy()).cuda()
            dyr, dyi = torch.empty_like(dxr), torch.empty_like(dxi)
        M.dspmv_complex_dev(dA, dxr.data_ptr(), dxi.data_ptr(), dyr.data_ptr(), dyi.data_ptr(), 1)
        ctx.synchronize()
        out = dyr.cpu().numpy(), dyi.cpu().numpy()
        dA.close()
        return out

    parts = _run_ranks(P, rank_fn)
    rr, ri = O.spmv_complex(A, xr, xi, 1)
    assert bits_equal(np.concatenate([p[0] for p in parts]), rr)
    assert bits_equal(np.concatenate([p[1] for p in parts]), ri)


@pytest.mark.parametrize("variant", [0, 1], ids=["auto_one_reduction", "classic"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("K", [2, 4])
def test_sharded_cg_several_ranks(P, K, variant):
    """Sharded CG: by default (auto) more than one rank runs the one-reduction
    form (one allgather per iteration, the scalar step in the next update's
    prologue); variant 1 keeps the reference's two reductions."""
    A = synth.config_matrix(5, K, 16)
    xt = synth.config_vector(5, A.nrows, K)
    b = O.spmv(A, xt, 1)
    bounds = M.partition_rows(A.indptr, A.nrows, P)
    cfg = M.SolverConfig(rel_tol=1e-22, max_iters=300, cg_variant=variant, check_every=5)

    def rank_fn(r, comm, ctx):
        dA = M.DistCsr.from_global(comm, A, K, bounds=bounds)
        res = M.dsolve_cg(dA, b[dA.row_begin:dA.row_end], cfg)
        dA.close()
        return res

    parts = _run_ranks(P, rank_fn)
    single = M.solve_cg(M.CsrOperator(M.DeviceCsr(A, K)), b, cfg)
    h0 = parts[0].report.residual_history
    for p in parts[1:]:  # every rank took the same decisions on the same numbers
        assert p.report.residual_history == h0 and p.report.iterations == parts[0].report.iterations
    assert parts[0].report.status == single.report.status
    assert abs(parts[0].report.iterations - single.report.iterations) <= 1
    x = np.concatenate([p.x for p in parts])
    assert np.allclose(x[:, 0], xt[:, 0], atol=1e-12)
    assert parts[0].report.final_true_residual <= 10 * single.report.final_true_residual + 1e-30


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_one_reduction_cg_x0_breakdown_and_max_iterations(P):
    """One-reduction sharded CG (the default over several ranks): an initial
    guess (r0 = b - A x0 through the halo exchange), MaxIterations with an odd
    iteration count and odd polling interval (both state parities), and the
    reference's breakdown report -- every rank with the same report."""
    K = 2
    A = synth.config_matrix(5, K, 12)
    xt = synth.config_vector(5, A.nrows, K)
    b = O.spmv(A, xt, 1)
    bounds = M.partition_rows(A.indptr, A.nrows, P)
    x0 = (0.5 * xt[:, 0]).tolist()

    def rank_fn(r, comm, ctx):
        dA = M.DistCsr.from_global(comm, A, K, bounds=bounds)
        lo, hi = dA.row_begin, dA.row_end
        a = M.dsolve_cg(dA, b[lo:hi], M.SolverConfig(rel_tol=1e-22, max_iters=300, x0=x0, check_every=3))
        m = M.dsolve_cg(dA, b[lo:hi], M.SolverConfig(rel_tol=1e-30, max_iters=7, check_every=3))
        dA.close()
        return a, m

    parts = _run_ranks(P, rank_fn)
    single = M.solve_cg(M.CsrOperator(M.DeviceCsr(A, K)), b, M.SolverConfig(rel_tol=1e-22, max_iters=300, x0=x0))
    a0, m0 = parts[0]
    for a, m in parts[1:]:
        assert a.report.residual_history == a0.report.residual_history
        assert m.report.residual_history == m0.report.residual_history
    assert a0.report.status == single.report.status == M.SolverStatus.Converged
    assert abs(a0.report.iterations - single.report.iterations) <= 1
    assert abs(a0.report.residual_history[0] - single.report.residual_history[0]) <= 1e-12 * single.report.residual_history[0]
    x = np.concatenate([p[0].x for p in parts])
    assert np.allclose(x[:, 0], xt[:, 0], atol=1e-12)
    assert m0.report.status == M.SolverStatus.MaxIterations and m0.report.iterations == 7
    assert len(m0.report.residual_history) == 8

    # skew-symmetric 2x2 blocks: <p, Ap> = 0 at the first step (test_krylov.cpp:193-211)
    n = 8
    S = csr(n, n, [[i ^ 1] for i in range(n)], 2,
            planes=np.array([[1.0 if i % 2 == 0 else -1.0 for i in range(n)], [0.0] * n]))
    sb = M.partition_rows(S.indptr, S.nrows, P)
    ones = np.zeros((n, 2))
    ones[:, 0] = 1.0

    def rank_bd(r, comm, ctx):
        dS = M.DistCsr.from_global(comm, S, 2, bounds=sb)
        res = M.dsolve_cg(dS, ones[dS.row_begin:dS.row_end], M.SolverConfig())
        dS.close()
        return res.report

    for rep in _run_ranks(P, rank_bd):
        assert rep.status == M.SolverStatus.Breakdown and rep.iterations == 0
        assert rep.detail == "cg: <p, Ap> vanished" and len(rep.residual_history) == 1


# ---- row-sharded solve() for the other Krylov methods (mpsg_dsolve) ----------------
@pytest.mark.parametrize("method", ["cg", "cgs", "bicgstab", "gpbicg"])
def test_one_rank_dsolve_equals_single_gpu_bits(ctx, method):
    """One rank: the sharded driver is the single-GPU driver plus a one-rank
    allgather -> identical bits, in both dot orders."""
    from tests.util import krylov_system

    A, b = krylov_system(200, 3, seed=4, symmetric=method == "cg", density=0.04)
    for exact in (True, False):
        cfg = M.SolverConfig(method=M.parse_method(method), rel_tol=1e-40, max_iters=150, exact_dots=exact)
        single = M.solve(M.CsrOperator(M.DeviceCsr(A, 3, ctx=ctx)), b, cfg)
        comm = M.Comm(ctx, 1, 0)
        dA = M.DistCsr.from_global(comm, A, 3)
        dist = M.dsolve(dA, b, cfg)
        assert dist.report.residual_history == single.report.residual_history
        assert bits_equal(dist.x, single.x) and dist.report.status == single.report.status
        dA.close()
        comm.close()
        if exact:  # and, with sequential dots, the reference's solve() itself (C restatement)
            ref = O.solve(A, b, method, rel_tol=1e-40, max_iters=150)
            assert bits_equal(np.array(dist.report.residual_history), ref["history"])
            assert bits_equal(dist.x, ref["x"])


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("method", ["cgs", "bicgstab", "gpbicg", "cg"])
def test_sharded_solvers_several_ranks(P, method):
    K = 4 if method in ("bicgstab", "cg") else 2
    A = synth.config_matrix(5, K, 14)
    xt = synth.config_vector(5, A.nrows, K)
    b = O.spmv(A, xt, 1)
    bounds = M.partition_rows(A.indptr, A.nrows, P)
    cfg = M.SolverConfig(method=M.parse_method(method), rel_tol=1e-22, max_iters=300)

    def rank_fn(r, comm, ctx):
        dA = M.DistCsr.from_global(comm, A, K, bounds=bounds)
        res = M.dsolve(dA, b[dA.row_begin:dA.row_end], cfg)
        dA.close()
        return res

    parts = _run_ranks(P, rank_fn)
    single = M.solve(M.CsrOperator(M.DeviceCsr(A, K)), b, cfg)
    h0 = parts[0].report.residual_history
    for p in parts[1:]:  # every rank took the same decisions on the same numbers
        assert p.report.residual_history == h0 and p.report.iterations == parts[0].report.iterations
    assert parts[0].report.status == single.report.status == M.SolverStatus.Converged
    assert abs(parts[0].report.iterations - single.report.iterations) <= max(2, single.report.iterations // 20)
    x = np.concatenate([p.x for p in parts])
    assert np.allclose(x[:, 0], xt[:, 0], atol=1e-12)
    assert parts[0].report.final_true_residual <= 1e-22 * parts[0].report.rhs_norm * 10


def test_dsolve_rejects_bicg(ctx):
    A = synth.config_matrix(5, 2, 6)
    b = O.spmv(A, synth.config_vector(5, A.nrows, 2), 1)
    comm = M.Comm(ctx, 1, 0)
    dA = M.DistCsr.from_global(comm, A, 2)
    with pytest.raises(M.MpsgError, match="row-sharded"):
        M.dsolve(dA, b, M.SolverConfig(method=M.KrylovMethod.BiCG))
    dA.close()
    comm.close()


@pytest.mark.parametrize("P,bad", [(2, 0), (3, 1), (3, 2)])
def test_failing_rank_fails_every_rank_without_hanging(P, bad):
    """One rank's local upload fails (a column index out of range): every rank
    gets an error from the collective setup instead of blocking in it."""
    import threading

    A = synth.config_matrix(5, 2, 10)
    bounds = M.partition_rows(A.indptr, A.nrows, P)
    ctxs = [M.Context(0) for _ in range(P)]
    comms = M.Comm.local_group(ctxs)
    errs = [None] * P

    def body(r):
        Al = M.shard_rows(A, int(bounds[r]), int(bounds[r + 1]))
        if r == bad:
            Al.indices = Al.indices.copy()
            Al.indices[0] = A.nrows + 7  # out of range
        try:
            d = M.DistCsr(comms[r], Al, 2, A.nrows, int(bounds[r]), int(bounds[r + 1]))
            d.close()
        except Exception as e:  # noqa: BLE001
            errs[r] = str(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts), "a rank hung in the setup collective"
    assert all(e is not None for e in errs), errs
    assert f"rank {bad} failed" in errs[(bad + 1) % P]
    for c in comms:
        c.close()
    for c in ctxs:
        c.close()
