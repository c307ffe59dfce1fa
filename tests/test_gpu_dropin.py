"""The C++ drop-in (include/mps/gpu.hpp) against the unmodified reference.

oracle/_ref/dropin_test is tests/cpp/dropin_test.cpp compiled with the
reference headers (make -C oracle dropin, in the build container where
/root/reference exists; the binary travels to the GPU box).  It checks
mps::gpu::spmv / spmv_complex bit-for-bit against mps::spmv / spmv_complex,
runs the reference's own solve_cg over a GpuCsrOperator and the device CG.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference sources absent")
def test_dropin_header_compiles_against_reference():
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_against_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs the reference sources at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    out = r.stdout
    print(out)
    assert "FAIL" not in out, out
    assert r.returncode == 0, out + r.stderr
    assert out.count("PASS") >= 40
