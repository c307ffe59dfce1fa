#!/usr/bin/env python
"""FAST-order accuracy under adversarial inputs (development probe): long QD/TD
rows (config 4 shape), a wide exponent range, and heavy cancellation; worst
|y - y_ref| / (4 rowlen u sum|a||x|) against the reference lanes-off order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2412_17510_b200 as M  # noqa: E402
import synth  # noqa: E402
from tests.util import bound_ok  # noqa: E402

ctx = M.Context(0)
tag = os.environ.get("MPSG_LIB", "default")[-10:]
rng = np.random.default_rng(1)
for K in (4, 3):
    # config-4 shape, long rows up to 20000 (long_fast chains + partial combine)
    A = synth.config_matrix(4, K, 60000, 20000.0, 1.8)
    x = synth.config_vector(4, A.nrows, K)
    y = M.spmv(M.DeviceCsr(A, K, ctx=ctx), x, M.ORDER_FAST)
    print(f"{tag} K={K} power-law long rows: ok,worst = {bound_ok(A, x, y, O.spmv(A, x, 0), K)}", flush=True)
    # wide exponent range: scale every value by 2^U[-60, 60]
    B = synth.config_matrix(2, K, 50000, 48.0)
    sc = np.exp2(rng.integers(-60, 61, B.planes.shape[1])).astype(float)
    B.planes *= sc[None, :]
    xb = synth.config_vector(2, B.nrows, K) * np.exp2(rng.integers(-60, 61, B.nrows)).astype(float)[:, None]
    y = M.spmv(M.DeviceCsr(B, K, ctx=ctx), xb, M.ORDER_FAST)
    print(f"{tag} K={K} wide exponents: ok,worst = {bound_ok(B, xb, y, O.spmv(B, xb, 0), K)}", flush=True)
    # cancellation: rows whose terms sum to ~0 (pairs a, -a against the same x)
    C = synth.config_matrix(2, K, 50000, 48.0)
    C.planes[:, 1::2] = -C.planes[:, 0::2][:, : C.planes[:, 1::2].shape[1]]
    xc = synth.config_vector(2, C.nrows, K)
    y = M.spmv(M.DeviceCsr(C, K, ctx=ctx), xc, M.ORDER_FAST)
    print(f"{tag} K={K} paired cancellation: ok,worst = {bound_ok(C, xc, y, O.spmv(C, xc, 0), K)}", flush=True)
