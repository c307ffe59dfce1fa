"""Generate tests/golden/*.npz from the REAL reference (oracle/_ref/libmpsref.so,
compiled from /root/reference by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py            # everything except full-size CG
    python tests/golden/make_golden.py --cg-full  # + 500-iteration config-5 CG (slow)

The fixtures pin both the C restatement (oracle/mpsoracle.c) and the CUDA path
on hosts where the reference sources are absent (the GPU box).  Inputs are
regenerated at test time from the seeded generators in synth/ (or the
operands stored here), so only outputs / checksums are stored.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synth  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# Small instances of the five configs (cfg, p1, p2, p3) used for full-vector pins.
SMALL = {
    "cfg1": (1, 16, 0.0, 0.0),
    "cfg2": (2, 600, 32.0, 0.0),
    "cfg3": (3, 300, 32.0, 0.0),
    "cfg4": (4, 3000, 700.0, 1.8),
    "cfg5": (5, 6, 0.0, 0.0),
}
# Full BASELINE.json instances pinned by checksum: (name, cfg, K list)
FULL = [("cfg1", 1, [2]), ("cfg2", 2, [3, 4]), ("cfg3", 3, [2, 4]), ("cfg4", 4, [2]), ("cfg5", 5, [2, 4])]


def arith(rng_seed=7, n=400):
    out = {}
    rng = np.random.default_rng(rng_seed)
    for K in (2, 3, 4):
        a = synth.vector(synth.VAL_NORMAL, n, K, seed=101 + K)
        b = synth.vector(synth.VAL_NORMAL, n, K, seed=201 + K)
        a *= rng.uniform(0.5, 8.0, size=(n, 1))  # exact power-free scaling keeps lower parts small
        a[: n // 8] = np.round(a[: n // 8, :1]) * np.eye(1, K)  # integer-valued, zero tails
        b[n // 4 : n // 4 + n // 8] = -b[n // 4 : n // 4 + n // 8]
        out[f"K{K}_a"], out[f"K{K}_b"] = a, b
        for op in ("add", "mul", "sub", "div"):
            out[f"K{K}_{op}"] = np.array([O.ref_mc_op(op, K, a[i], b[i]) for i in range(n)])
        out[f"K{K}_mul_d"] = np.array([O.ref_mc_op("mul_d", K, a[i], b[i, 0]) for i in range(n)])
        aa = np.abs(a) * np.sign(a[:, :1]) * np.sign(a[:, :1])  # positive leading component
        aa = np.where(a[:, :1] < 0, -a, a)
        out[f"K{K}_sqrt_a"] = aa
        out[f"K{K}_sqrt"] = np.array([O.ref_mc_op("sqrt", K, aa[i]) for i in range(n)])
    return out


def spmv_small():
    out = {}
    # worked 5x5 example (test_kernels.cpp:99-138): A * [1..5] = [7,-14,15,-22,40]
    ex = O.ref_fixture("example5x5")
    for K in (2, 3, 4):
        A = _widen(ex, K)
        x = np.zeros((5, K))
        x[:, 0] = np.arange(1, 6)
        for order in (0, 1):
            out[f"ex5_K{K}_o{order}"] = O.ref_spmv(A, x, order)
    for name, (cfg, p1, p2, p3) in SMALL.items():
        for K in (2, 3, 4):
            A = synth.config_matrix(cfg, K, p1, p2, p3, seed=0)
            if cfg == 3:
                xr, xi = synth.config_vector(3, A.nrows, K)
                for order in (0, 1):
                    yr, yi = O.ref_spmv_complex(A, xr, xi, order)
                    out[f"{name}_K{K}_o{order}_re"], out[f"{name}_K{K}_o{order}_im"] = yr, yi
            else:
                x = synth.config_vector(cfg, A.nrows, K)
                for order in (0, 1):
                    out[f"{name}_K{K}_o{order}"] = O.ref_spmv(A, x, order)
    # reference stand-in fixtures with the reference's make_vector (bench.hpp:78-111)
    tub = O.ref_fixture("tub1000")
    for K in (2, 3, 4):
        A = _widen(tub, K)
        v = O.ref_make_vector(K, tub.nrows)
        out[f"make_vector_K{K}"] = v
        for order in (0, 1):
            out[f"tub1000_K{K}_o{order}"] = O.ref_spmv(A, v, order)
    qre, qim = O.ref_fixture("qc324_re"), O.ref_fixture("qc324_im")
    for K in (2, 4):
        A = _complex(qre, qim, K)
        vr, vi = O.ref_make_complex_vector(K, qre.nrows)
        out[f"make_cvector_K{K}_re"], out[f"make_cvector_K{K}_im"] = vr, vi
        for order in (0, 1):
            yr, yi = O.ref_spmv_complex(A, vr, vi, order)
            out[f"qc324_K{K}_o{order}_re"], out[f"qc324_K{K}_o{order}_im"] = yr, yi
    return out


def _widen(m, K):
    from types import SimpleNamespace

    planes = np.zeros((K, m.nnz))
    planes[0] = m.planes[0]
    return SimpleNamespace(nrows=m.nrows, ncols=m.ncols, indptr=m.indptr, indices=m.indices, planes=planes, K=K)


def _complex(re, im, K):
    from types import SimpleNamespace

    assert np.array_equal(re.indptr, im.indptr) and np.array_equal(re.indices, im.indices)
    planes = np.zeros((2 * K, re.nnz))
    planes[0] = re.planes[0]
    planes[K] = im.planes[0]
    return SimpleNamespace(nrows=re.nrows, ncols=re.ncols, indptr=re.indptr, indices=re.indices, planes=planes,
                           K=K)


def spmv_full():
    out = {}
    for name, cfg, Ks in FULL:
        for K in Ks:
            t = time.time()
            A = synth.config_matrix(cfg, K)
            x = synth.config_vector(cfg, A.nrows, K)
            orders = (0, 1)
            for order in orders:
                if cfg == 3:
                    Ah, xh, yh = O.RefComplex(A, K), O.RefCVec(*x), O.RefCVec(K=K)
                    rc = O.ref().ref_spmv_complex(Ah.h, xh.h, order, 8, yh.h)
                    assert rc == 0
                    out[f"{name}_K{K}_o{order}"] = np.uint64(yh.checksum())
                else:
                    Ah, xh, yh = O.RefCsr(A, K), O.RefVec(x), O.RefVec(K=K)
                    O.ref_spmv_h(Ah, xh, yh, order, 8)
                    out[f"{name}_K{K}_o{order}"] = np.uint64(yh.checksum())
                    if cfg == 5 and order == 1:
                        # b = A x_true, the CG right-hand side (LANE4, CsrOperator default)
                        np.save(os.path.join("/tmp", f"cfg5_b_K{K}.npy"), yh.read())
            out[f"{name}_K{K}_nnz"] = np.int64(A.nnz)
            print(f"  full {name} K={K}: {time.time() - t:.1f}s", flush=True)
    return out


def cg_small():
    out = {}
    for K in (2, 3, 4):
        A = synth.config_matrix(5, K, p1=10)
        xt = synth.config_vector(5, A.nrows, K)
        b = O.ref_spmv(A, xt, 1)
        r = O.ref_cg(A, b, 1, rel_tol=1e-30, max_iters=80)
        out[f"cg5s_K{K}_history"] = r["history"]
        out[f"cg5s_K{K}_x"] = r["x"]
        out[f"cg5s_K{K}_meta"] = np.array([r["iterations"], r["status"], r["rhs_norm"], r["final_true_residual"]])
        # converging run (default tolerance)
        r2 = O.ref_cg(A, b, 1, rel_tol=1e-20, max_iters=400)
        out[f"cg5c_K{K}_history"] = r2["history"]
        out[f"cg5c_K{K}_meta"] = np.array([r2["iterations"], r2["status"], r2["rhs_norm"], r2["final_true_residual"]])
    # diag(1..40), QD (test_krylov.cpp:94-116)
    from types import SimpleNamespace

    k = 40
    A = SimpleNamespace(nrows=k, ncols=k, indptr=np.arange(k + 1), indices=np.arange(k),
                        planes=np.vstack([np.arange(1, k + 1, dtype=float), np.zeros((3, k))]))
    b = synth.vector(synth.VAL_UNIFORM0, k, 4, seed=40)
    b[:, 0] = np.abs(b[:, 0]) + 0.25
    r = O.ref_cg(A, b, 1, rel_tol=1e-50)
    out["diag40_b"] = b
    out["diag40_meta"] = np.array([r["iterations"], r["status"], r["rhs_norm"], r["final_true_residual"]])
    out["diag40_history"] = r["history"]
    return out


def cg_full():
    out = {}
    for K in (2, 4):
        A = synth.config_matrix(5, K)
        xt = synth.config_vector(5, A.nrows, K)
        b = O.ref_spmv(A, xt, 1, threads=8)
        t = time.time()
        r = O.ref_cg(A, b, 1, threads=8, rel_tol=1e-30, max_iters=500)
        print(f"  full CG K={K}: {time.time() - t:.0f}s", flush=True)
        out[f"cg5_K{K}_history"] = r["history"]
        out[f"cg5_K{K}_meta"] = np.array([r["iterations"], r["status"], r["rhs_norm"], r["final_true_residual"]])
        out[f"cg5_K{K}_b_checksum"] = np.uint64(O.checksum(b))
    return out


def mixed_sptmv():
    """Mixed-mode SpMV and (complex) sptmv outputs from the real reference."""
    from tests.util import mixed_of

    cases = {"cfg2": (2, 600, 32.0, 0.0), "cfg4": (4, 3000, 700.0, 1.8)}
    out = {}
    for name, K, order in (("cfg2", 4, 1), ("cfg4", 2, 0)):
        c = cases[name]
        A = mixed_of(synth.config_matrix(c[0], K, *c[1:]))
        x = synth.config_vector(c[0], A.nrows, K)
        out[f"mixed_{name}_K{K}_o{order}"] = O.ref_spmv(A, x, order, mixed=True)
    for name, K, mixed in (("cfg2", 3, False), ("cfg4", 2, True)):
        c = cases[name]
        A = synth.config_matrix(c[0], K, *c[1:])
        if mixed:
            A = mixed_of(A)
        v = synth.config_vector(c[0], A.nrows, K)
        out[f"sptmv_{'mixed_' if mixed else ''}{name}_K{K}"] = O.ref_sptmv(A, v, 1, threads=1, mixed=mixed)
    A = synth.config_matrix(3, 4, 300, 24.0)
    vr, vi = synth.config_vector(3, A.nrows, 4)
    yr, yi = O.ref_sptmv_complex(A, vr, vi, 1, threads=1, conjugate=True)
    out["csptmv_K4_conj_re"], out["csptmv_K4_conj_im"] = yr, yi
    return out


def krylov_small():
    """The reference solve() (all five methods) on tests.util.krylov_cases()."""
    from tests.util import krylov_cases

    out = {}
    for name, A, b, m, kw in krylov_cases():
        r = O.ref_solve(A, b, m, **kw)
        out[f"{name}_history"] = r["history"]
        out[f"{name}_x"] = r["x"]
        out[f"{name}_meta"] = np.array([r["iterations"], r["status"], r["rhs_norm"], r["final_true_residual"]])
        out[f"{name}_detail"] = np.array(r["detail"])
    return out


def krylov_mixed():
    """The reference solve() over CsrOperator<double> (Mixed mode)."""
    from tests.util import krylov_mixed_cases

    out = {}
    for name, A, b, m, kw in krylov_mixed_cases():
        r = O.ref_solve(A, b, m, mixed=True, **kw)
        out[f"{name}_history"] = r["history"]
        out[f"{name}_x"] = r["x"]
        out[f"{name}_meta"] = np.array([r["iterations"], r["status"], r["rhs_norm"], r["final_true_residual"]])
        out[f"{name}_detail"] = np.array(r["detail"])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cg-full", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    assert O.ref_available(), "build the reference first: make -C oracle ref"
    jobs = {"arith": arith, "spmv_small": spmv_small, "spmv_full": spmv_full, "cg_small": cg_small,
            "mixed_sptmv": mixed_sptmv, "krylov_small": krylov_small, "krylov_mixed": krylov_mixed}
    if a.cg_full:
        jobs = {"cg_full": cg_full}
    for name, fn in jobs.items():
        if a.only and name not in a.only.split(","):
            continue
        t = time.time()
        data = fn()
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
        print(f"{name}: {len(data)} arrays, {time.time() - t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
