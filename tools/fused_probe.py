#!/usr/bin/env python
"""FAST-order accuracy probe: worst |y - y_ref| / (4 rowlen u sum|a||x|) over
all rows of configs 2 / 3-real-part / 5 against the reference order (oracle),
for the library selected by MPSG_LIB; plus timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2412_17510_b200 as M  # noqa: E402
import synth  # noqa: E402
from tests.util import bound_ok  # noqa: E402

ctx = M.Context(0)
tag = os.environ.get("MPSG_LIB", "default")[-12:]
for cfg, K, kw in ((2, 4, {}), (2, 3, {}), (5, 4, {}), (2, 4, {"p1": 200000, "p2": 64.0})):
    A = synth.config_matrix(cfg, K, **kw)
    x = synth.config_vector(cfg, A.nrows, K)
    dA = M.DeviceCsr(A, K, ctx=ctx)
    y = M.spmv(dA, x, M.ORDER_FAST)
    ref = O.spmv(A, x, 0)
    ok, worst = bound_ok(A, x, y, ref, K)
    same = np.mean(np.all(y == ref, axis=1))
    print(f"{tag} cfg{cfg} K={K} {kw}: bound ok={ok} worst ratio={worst:.3g} rows bit-equal to SCALAR={same:.3f}",
          flush=True)
    # adversarial: alternate signs so rows cancel heavily
    B = synth.config_matrix(cfg, K, **kw)
    B.planes[:, ::2] *= -1.0
    xb = np.abs(x)
    yb = M.spmv(M.DeviceCsr(B, K, ctx=ctx), xb, M.ORDER_FAST)
    ok2, worst2 = bound_ok(B, xb, yb, O.spmv(B, xb, 0), K)
    print(f"{tag}   cancelling: bound ok={ok2} worst ratio={worst2:.3g}", flush=True)
