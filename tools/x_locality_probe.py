#!/usr/bin/env python
"""How much of config 4's time is x-gather L2 misses?  Times the FAST SpMV on
the real matrix and on copies whose column indices are folded into the first
n/F columns (same row structure and matrix bytes, x working set / F)."""
import os
import statistics
import sys
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_17510_b200 as M  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = M.Context(0)
ctx.set_stream(stream.cuda_stream)
f1 = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
f2 = torch.ones(64 * 1024 * 1024, dtype=torch.int32, device=dev)
acc = torch.zeros(1, dtype=torch.int64, device=dev)
K = 2
A = synth.config_matrix(4, K)
x = synth.config_vector(4, A.nrows, K)
mixed = len(sys.argv) > 1 and sys.argv[1] == "mixed"
for F in [int(f) for f in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,16,64").split(",")]:
    if F == 1:
        B = A
    else:
        ind = (A.indices % (A.ncols // F)).astype(np.int64)
        B = SimpleNamespace(nrows=A.nrows, ncols=A.ncols, indptr=A.indptr, indices=ind, planes=A.planes, nnz=A.nnz)
    planes = B.planes[:1] if mixed else B.planes
    Bv = SimpleNamespace(nrows=B.nrows, ncols=B.ncols, indptr=B.indptr, indices=B.indices, planes=planes, nnz=B.nnz)
    dA = M.DeviceCsr(Bv, K, ctx=ctx, mixed=mixed)
    dx = torch.from_numpy(x).to(dev)
    dy = torch.empty((A.nrows, K), dtype=torch.float64, device=dev)
    step = lambda: M.spmv_dev(dA, dx.data_ptr(), dy.data_ptr(), M.ORDER_FAST, stream.cuda_stream)  # noqa
    for _ in range(3):
        step()
    ms = []
    for _ in range(10):
        torch.cuda.synchronize()
        f1.zero_()
        acc += f2.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    med = statistics.median(ms)
    print(f"{os.environ.get('MPSG_LIB', 'default')[-12:]} {'mixed' if mixed else 'pure'} fold F={F}: x working set {A.ncols // F * K * 8 / 2**20:.0f} MB, "
          f"{med * 1e3:.1f} us, {A.nnz / med / 1e6:.1f} Gnnz/s", flush=True)
    del dA
