"""CPU: pin the C restatement (oracle/mpsoracle.c) against the reference's
golden vectors (tests/golden/, generated from the compiled reference by
tests/golden/make_golden.py) and, where the reference was built here, against
the live reference itself."""
import numpy as np
import pytest

import oracle as O
import synth
from tests.util import bits_equal, golden, widen

SMALL = {"cfg1": (1, 16, 0.0, 0.0), "cfg2": (2, 600, 32.0, 0.0), "cfg3": (3, 300, 32.0, 0.0),
         "cfg4": (4, 3000, 700.0, 1.8), "cfg5": (5, 6, 0.0, 0.0)}


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("op", ["add", "mul", "sub", "div", "mul_d", "sqrt"])
def test_arith_matches_reference_bits(K, op):
    g = golden("arith")
    a, b = g[f"K{K}_a"], g[f"K{K}_b"]
    if op == "sqrt":
        a = g[f"K{K}_sqrt_a"]
        got = np.array([O.mc_op("sqrt", K, ai) for ai in a])
    elif op == "mul_d":
        got = np.array([O.mc_op("mul_d", K, a[i], b[i, 0]) for i in range(len(a))])
    else:
        got = np.array([O.mc_op(op, K, a[i], b[i]) for i in range(len(a))])
    assert bits_equal(got, g[f"K{K}_{op}"])


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("order", [0, 1])
def test_worked_example_exact(K, order):
    # test_kernels.cpp:99-138: A * [1..5] = [7, -14, 15, -22, 40] exactly
    A = widen(_example5x5(), K)
    x = np.zeros((5, K))
    x[:, 0] = np.arange(1, 6)
    y = O.spmv(A, x, order)
    assert list(y[:, 0]) == [7.0, -14.0, 15.0, -22.0, 40.0]
    assert np.all(y[:, 1:] == 0.0)
    assert bits_equal(y, golden("spmv_small")[f"ex5_K{K}_o{order}"])


def _example5x5():
    from types import SimpleNamespace

    return SimpleNamespace(nrows=5, ncols=5, indptr=np.array([0, 2, 4, 5, 7, 8]),
                           indices=np.array([0, 2, 1, 4, 2, 0, 3, 4]),
                           planes=np.array([[1.0, 2, 3, -4, 5, 6, -7, 8]]), nnz=8)


@pytest.mark.parametrize("name", list(SMALL))
@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("order", [0, 1])
def test_small_configs_match_reference(name, K, order):
    cfg, p1, p2, p3 = SMALL[name]
    A = synth.config_matrix(cfg, K, p1, p2, p3)
    g = golden("spmv_small")
    if cfg == 3:
        xr, xi = synth.config_vector(3, A.nrows, K)
        yr, yi = O.spmv_complex(A, xr, xi, order)
        assert bits_equal(yr, g[f"{name}_K{K}_o{order}_re"])
        assert bits_equal(yi, g[f"{name}_K{K}_o{order}_im"])
    else:
        x = synth.config_vector(cfg, A.nrows, K)
        assert bits_equal(O.spmv(A, x, order), g[f"{name}_K{K}_o{order}"])


def test_lane_order_differs_from_scalar_on_random_rows():
    # the two reference orders are distinct on random data: both must be offered
    g = golden("spmv_small")
    assert not bits_equal(g["cfg2_K4_o0"], g["cfg2_K4_o1"])


@pytest.mark.parametrize("K", [2, 3, 4])
def test_reference_fixtures_tub1000(K):
    g = golden("spmv_small")
    # tub1000 stand-in (fixtures.hpp:21-35) rebuilt here from its closed form
    A = widen(_tub1000(), K)
    v = g[f"make_vector_K{K}"]
    for order in (0, 1):
        assert bits_equal(O.spmv(A, v, order), g[f"tub1000_K{K}_o{order}"])


def _tub1000():
    from types import SimpleNamespace

    n = 1000
    rows, vals = [], []
    for i in range(n):
        r, v = [], []
        if i >= 1:
            r.append(i - 1), v.append(-(1.0 + 0.125 * ((3 * i) % 7)))
        r.append(i), v.append(6.0 + 0.25 * ((7 * i) % 13))
        if i + 1 < n:
            r.append(i + 1), v.append(1.0 + 0.125 * ((5 * i) % 11))
        if i + 2 < n:
            r.append(i + 2), v.append(0.5 + 0.125 * ((2 * i) % 5))
        rows.append(r)
        vals.extend(v)
    indptr = np.cumsum([0] + [len(r) for r in rows])
    return SimpleNamespace(nrows=n, ncols=n, indptr=indptr, indices=np.array([c for r in rows for c in r]),
                           planes=np.array([vals]), nnz=len(vals))


@pytest.mark.parametrize("K", [2, 4])
def test_reference_fixture_qc324_complex(K):
    g = golden("spmv_small")
    if not O.ref_available():
        pytest.skip("qc324 stand-in structure is rebuilt only from the reference fixture")
    qre, qim = O.ref_fixture("qc324_re"), O.ref_fixture("qc324_im")
    from types import SimpleNamespace

    planes = np.zeros((2 * K, qre.nnz))
    planes[0], planes[K] = qre.planes[0], qim.planes[0]
    A = SimpleNamespace(nrows=qre.nrows, ncols=qre.ncols, indptr=qre.indptr, indices=qre.indices, planes=planes)
    vr, vi = g[f"make_cvector_K{K}_re"], g[f"make_cvector_K{K}_im"]
    for order in (0, 1):
        yr, yi = O.spmv_complex(A, vr, vi, order)
        assert bits_equal(yr, g[f"qc324_K{K}_o{order}_re"]) and bits_equal(yi, g[f"qc324_K{K}_o{order}_im"])


@pytest.mark.parametrize("K", [2, 3, 4])
def test_cg_small_matches_reference(K):
    g = golden("cg_small")
    A = synth.config_matrix(5, K, p1=10)
    xt = synth.config_vector(5, A.nrows, K)
    b = O.spmv(A, xt, 1)
    r = O.cg(A, b, 1, rel_tol=1e-30, max_iters=80)
    assert np.array_equal(r["history"], g[f"cg5s_K{K}_history"])
    assert bits_equal(r["x"], g[f"cg5s_K{K}_x"])
    meta = g[f"cg5s_K{K}_meta"]
    assert r["iterations"] == meta[0] and r["status"] == meta[1]
    assert r["rhs_norm"] == meta[2] and r["final_true_residual"] == meta[3]


def test_cg_diag40_qd():
    # test_krylov.cpp:94-116: CG on diag(1..40) in QD converges within k+2 iterations
    g = golden("cg_small")
    from types import SimpleNamespace

    k = 40
    A = SimpleNamespace(nrows=k, ncols=k, indptr=np.arange(k + 1), indices=np.arange(k),
                        planes=np.vstack([np.arange(1, k + 1, dtype=float), np.zeros((3, k))]))
    r = O.cg(A, g["diag40_b"], 1, rel_tol=1e-50)
    assert r["status"] == 0 and r["iterations"] <= k + 2
    assert np.array_equal(r["history"], g["diag40_history"])


def test_cg_breakdown_on_skew_system():
    # test_krylov.cpp:193-211
    from types import SimpleNamespace

    A = SimpleNamespace(nrows=2, ncols=2, indptr=np.array([0, 1, 2]), indices=np.array([1, 0]),
                        planes=np.array([[1.0, -1.0], [0.0, 0.0]]))
    r = O.cg(A, np.array([[1.0, 0.0], [1.0, 0.0]]))
    assert r["status"] == 2 and r["iterations"] == 0 and len(r["history"]) == 1
    assert abs(r["final_true_residual"] - np.sqrt(2.0)) < 1e-15


def test_full_cfg1_checksum_matches_reference():
    g = golden("spmv_full")
    A = synth.config_matrix(1, 2)
    assert A.nnz == int(g["cfg1_K2_nnz"]) == 1_308_672
    x = synth.config_vector(1, A.nrows, 2)
    for order in (0, 1):
        assert O.checksum(O.spmv(A, x, order)) == int(g[f"cfg1_K2_o{order}"])


@pytest.mark.skipif(not O.ref_available(), reason="live reference not built on this host")
@pytest.mark.parametrize("K", [2, 3, 4])
def test_live_reference_random_matrices(K):
    # random_coo stand-ins (fixtures.hpp:166-185) with non-canonical vectors
    m = O.ref_fixture("random_coo", seed=0x6E61F002, a=300, b=300, c=4000)
    A = widen(m, K)
    x = synth.vector(synth.VAL_NORMAL, 300, K, seed=5)
    for order in (0, 1):
        assert bits_equal(O.spmv(A, x, order), O.ref_spmv(A, x, order))


# ---- Mixed mode and transposed products ----------------
from tests.util import mixed_of  # noqa: E402


@pytest.mark.parametrize("K", [2, 3, 4])
def test_mixed_and_sptmv_match_live_reference(K):
    if not O.ref_available():
        pytest.skip("reference not built here")
    A = synth.config_matrix(4, K, 1500, 400.0, 1.8)
    x = synth.config_vector(4, A.nrows, K)
    Am = mixed_of(A)
    for order in (0, 1):
        assert O.spmv(Am, x, order, mixed=True).tobytes() == O.ref_spmv(Am, x, order, mixed=True).tobytes()
        for threads in (1, 2, 5):
            # sptmv: lanes on/off give the same bits; thread count changes the merge order
            assert O.sptmv(A, x, threads).tobytes() == O.ref_sptmv(A, x, order, threads=threads).tobytes()
            assert (O.sptmv(Am, x, threads, mixed=True).tobytes() ==
                    O.ref_sptmv(Am, x, order, threads=threads, mixed=True).tobytes())
    C = synth.config_matrix(3, K, 150, 10.0)
    xr, xi = synth.config_vector(3, C.nrows, K)
    for mixed, MM in ((False, C), (True, mixed_of(C, cplx=True))):
        a = O.spmv_complex(MM, xr, xi, 1, mixed=mixed)
        b = O.ref_spmv_complex(MM, xr, xi, 1, mixed=mixed)
        assert all(p.tobytes() == q.tobytes() for p, q in zip(a, b))
        for conj in (False, True):
            a = O.sptmv_complex(MM, xr, xi, 1, conj, mixed)
            b = O.ref_sptmv_complex(MM, xr, xi, 0, 1, conj, mixed)
            assert all(p.tobytes() == q.tobytes() for p, q in zip(a, b))


def test_mixed_sptmv_goldens_pin_the_oracle():
    g = golden("mixed_sptmv")
    c = {"cfg2": (2, 600, 32.0, 0.0), "cfg4": (4, 3000, 700.0, 1.8)}
    A = mixed_of(synth.config_matrix(2, 4, *c["cfg2"][1:]))
    assert O.spmv(A, synth.config_vector(2, A.nrows, 4), 1, mixed=True).tobytes() == g["mixed_cfg2_K4_o1"].tobytes()
    A = synth.config_matrix(2, 3, *c["cfg2"][1:])
    assert O.sptmv(A, synth.config_vector(2, A.nrows, 3)).tobytes() == g["sptmv_cfg2_K3"].tobytes()
    A = synth.config_matrix(3, 4, 300, 24.0)
    vr, vi = synth.config_vector(3, A.nrows, 4)
    yr, yi = O.sptmv_complex(A, vr, vi, 1, True)
    assert yr.tobytes() == g["csptmv_K4_conj_re"].tobytes() and yi.tobytes() == g["csptmv_K4_conj_im"].tobytes()


def test_sptmv_single_thread_equals_spmv_of_transpose():
    # test_kernels.cpp:152-174 / acceptance check 6: sptmv(1 thread, lanes off) == spmv(A^T)
    from tests.util import transpose

    A = synth.config_matrix(2, 2, 700, 16.0)
    v = synth.config_vector(2, A.nrows, 2)
    assert O.sptmv(A, v).tobytes() == O.spmv(transpose(A), v, 0).tobytes()


# ---- Krylov solvers (krylov.hpp:238-606): the C restatement vs the reference ----
from tests.util import BREAKDOWN_CASES, krylov_cases  # noqa: E402

_KCASES = krylov_cases()


@pytest.mark.parametrize("case", _KCASES, ids=[c[0] for c in _KCASES])
def test_oracle_solvers_equal_reference_golden(case):
    """Every method, bit for bit: iterate, residual history, iteration count,
    status, detail text and final true residual (golden from the reference's
    own solve(), tests/golden/make_golden.py krylov_small)."""
    name, A, b, m, kw = case
    g = golden("krylov_small")
    r = O.solve(A, b, m, **kw)
    meta = g[f"{name}_meta"]
    assert bits_equal(r["history"], g[f"{name}_history"])
    assert bits_equal(r["x"], g[f"{name}_x"])
    assert (r["iterations"], r["status"]) == (int(meta[0]), int(meta[1]))
    assert bits_equal(np.array([r["rhs_norm"], r["final_true_residual"]]), meta[2:])
    assert r["detail"] == str(g[f"{name}_detail"])


def test_breakdown_cases_cover_every_exit():
    details = {d for _, _, _, d in BREAKDOWN_CASES}
    assert len(details) == len(BREAKDOWN_CASES)
    g = golden("krylov_small")
    for i, (m, _, _, d) in enumerate(BREAKDOWN_CASES):
        assert str(g[f"breakdown{i}_{m}_detail"]) == d
        assert int(g[f"breakdown{i}_{m}_meta"][1]) == 2  # SolverStatus::Breakdown


@pytest.mark.skipif(not O.ref_available(), reason="live reference not built on this host")
@pytest.mark.parametrize("m", O.METHODS)
@pytest.mark.parametrize("threads", [1, 4])
def test_oracle_solvers_equal_live_reference(m, threads):
    from tests.util import krylov_system

    A, b = krylov_system(50, 2, seed=17, symmetric=m == "cg", density=0.15)
    r1 = O.solve(A, b, m, threads=threads, order=0)
    r2 = O.ref_solve(A, b, m, threads=threads, order=0)
    assert bits_equal(r1["history"], r2["history"]) and bits_equal(r1["x"], r2["x"])
    assert (r1["iterations"], r1["status"], r1["detail"]) == (r2["iterations"], r2["status"], r2["detail"])


def test_oracle_solver_rejects_bad_config():
    A, b = krylov_cases()[0][1:3]
    with pytest.raises(ValueError):
        O.solve(A, b, "cg", rel_tol=0.0)
    with pytest.raises(ValueError):
        O.solve(A, b, "cg", max_iters=0)


# ---- Mixed-mode solve() (CsrOperator<double>, bench.cpp:550-557) --------------
from tests.util import krylov_mixed_cases  # noqa: E402

_MCASES = krylov_mixed_cases()


@pytest.mark.parametrize("case", _MCASES, ids=[c[0] for c in _MCASES])
def test_oracle_mixed_solvers_equal_reference_golden(case):
    name, A, b, m, kw = case
    g = golden("krylov_mixed")
    r = O.solve(A, b, m, mixed=True, **kw)
    meta = g[f"{name}_meta"]
    assert bits_equal(r["history"], g[f"{name}_history"])
    assert bits_equal(r["x"], g[f"{name}_x"])
    assert (r["iterations"], r["status"]) == (int(meta[0]), int(meta[1]))
    assert r["detail"] == str(g[f"{name}_detail"])
