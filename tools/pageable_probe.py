#!/usr/bin/env python
"""Host-pointer SpMV (mpsg_spmv) end to end with pageable numpy buffers (what
the C++ drop-in's std::vector gives) vs pinned buffers, config 2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_17510_b200 as M  # noqa: E402
import synth  # noqa: E402

ctx = M.Context(0)
for K in (4, 2):
    A = synth.config_matrix(2, K)
    x = synth.config_vector(2, A.nrows, K)
    dA = M.DeviceCsr(A, K, ctx=ctx)
    y = np.empty_like(x)
    hx = torch.from_numpy(x).pin_memory()
    hy = torch.empty(x.shape, dtype=torch.float64).pin_memory()
    for name, xp, yp in (("pageable", x.ctypes.data, y.ctypes.data), ("pinned", hx.data_ptr(), hy.data_ptr())):
        for _ in range(3):
            ctx.check(M.lib().mpsg_spmv(ctx.h, dA.h, 2, A.nrows, xp, yp))
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            ctx.check(M.lib().mpsg_spmv(ctx.h, dA.h, 2, A.nrows, xp, yp))
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[len(ts) // 2]
        print(f"K={K} {name}: {t * 1e3:.3f} ms = {A.nnz / t / 1e9:.1f} Gnnz/s", flush=True)
