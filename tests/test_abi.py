"""CPU-side checks of the C ABI (no GPU needed).

* libmpsg.so loads and exports every function include/mpsg.h declares;
* the host-only entry points (partition_rows, checksum) agree with the
  reference's definitions (kernels.hpp:63-80, bench.hpp:113-150) and with the
  C restatement in oracle/;
* device entry points fail loudly (status code, no fallback) without a GPU.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2412_17510_b200 as M
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "mpsg.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"MPSG_API\s+[^;(]*?\b(mpsg_\w+)\s*\(", src)))


def test_header_declares_expected_set():
    names = _declared()
    assert len(names) >= 18
    assert set(names) == set(M.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = M.lib()
    missing = [s for s in _declared() if not hasattr(L, s)]
    assert not missing, missing


def test_library_exports_nothing_undeclared():
    # -fvisibility=hidden: the only dynamic symbols are the declared ABI
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", M.LIB_PATH], capture_output=True, text=True).stdout
    ours = {ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-1].startswith("mpsg_")}
    assert ours == set(_declared())


def test_version_string():
    assert "sm_100a" in M.version()


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8, 13])
def test_partition_rows_matches_reference_rule(parts):
    A = synth.config_matrix(4, 2, 5000, 3000.0, 1.8)
    b = M.partition_rows(A.indptr, A.nrows, parts)
    total = int(A.indptr[-1])
    assert b[0] == 0 and b[-1] == A.nrows
    for t in range(1, parts):
        # bounds[t] = lower_bound(indptr, total*t/parts) (kernels.hpp:70-77)
        assert b[t] == np.searchsorted(A.indptr, total * t // parts, side="left")
    assert np.all(np.diff(b) >= 0)


def test_partition_rows_empty_matrix():
    b = M.partition_rows(np.zeros(1, np.int64), 0, 4)
    assert list(b) == [0, 0, 0, 0, 0]


@pytest.mark.parametrize("K", [2, 3, 4])
def test_checksum_matches_oracle_and_reference(K):
    v = synth.vector(synth.VAL_NORMAL, 1000, K, seed=7)
    h = M.checksum(v)
    assert h == O.checksum(v)
    if O.ref_available():
        assert h == O.RefVec(v).checksum()


def test_checksum_sensitivity():
    # bench.hpp checksum is sensitive to order, sign (incl. -0) and every component
    v = synth.vector(synth.VAL_NORMAL, 16, 2, seed=3)
    h = M.checksum(v)
    w = v.copy()
    w[[0, 1]] = w[[1, 0]]
    assert M.checksum(w) != h
    z = np.zeros((1, 2))
    nz = z.copy()
    nz[0, 0] = -0.0
    assert M.checksum(z) != M.checksum(nz)
    w = v.copy()
    w[5, 1] = np.nextafter(w[5, 1], np.inf)
    assert M.checksum(w) != h


def test_checksum_complex_combination():
    re_, im_ = synth.vector(synth.VAL_NORMAL, 50, 4, 1), synth.vector(synth.VAL_NORMAL, 50, 4, 2)
    P = 1099511628211
    want = ((M.checksum(re_) * P) & (2**64 - 1)) ^ M.checksum(im_)
    assert M.checksum_complex(re_, im_) == want


def test_device_calls_fail_loudly_without_gpu():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(M.MpsgError):
        M.Context(0)


def test_null_arguments_rejected():
    L = M.lib()
    assert L.mpsg_spmv(None, None, 0, 0, None, None) == M.E_ARG
    assert L.mpsg_cg(None, None, 0, 0, None, None, None, None, None, 0, None) == M.E_ARG
    assert L.mpsg_partition_rows(None, 0, 1, None) == M.E_ARG
    assert L.mpsg_last_error(None) == b"null context"


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of the ABI structs have the sizes the C compiler gives
    the declarations in include/mpsg.h (a field added on one side only would
    silently shift everything after it)."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "sizes.c"
    src.write_text('#include <stdio.h>\n#include "mpsg.h"\n'
                   'int main(void) { printf("%zu %zu %zu %zu\\n", sizeof(mpsg_cg_config), '
                   'sizeof(mpsg_solver_config), sizeof(mpsg_cg_report), sizeof(mpsg_csr_stats)); return 0; }\n')
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-I", os.path.join(root, "include"), "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert [int(v) for v in out] == [ctypes.sizeof(M._CgConfig), ctypes.sizeof(M._SolverConfig),
                                     ctypes.sizeof(M._CgReport), ctypes.sizeof(M.CsrStats)]


def test_solver_config_validates_the_cg_variant():
    for v in (0, 1, 2):
        M.SolverConfig(cg_variant=v).validate()
    with pytest.raises(ValueError, match="cg_variant"):
        M.SolverConfig(cg_variant=3).validate()
