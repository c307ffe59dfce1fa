#!/usr/bin/env python
"""e2e breakdown of the host-pointer SpMV (mpsg_spmv) on config 2 QD: the call
itself vs its pieces (H2D, device SpMV, D2H), L2 flushed before each."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_17510_b200 as M  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = M.Context(0)
ctx.set_stream(stream.cuda_stream)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
A = synth.config_matrix(2, K)
x = synth.config_vector(2, A.nrows, K)
dA = M.DeviceCsr(A, K, ctx=ctx)
n = A.nrows
hx = torch.from_numpy(x).pin_memory()
hy = torch.empty((n, K), dtype=torch.float64).pin_memory()
dx = torch.empty((n, K), dtype=torch.float64, device=dev)
dy = torch.empty((n, K), dtype=torch.float64, device=dev)
f1 = torch.empty(64 * 2**20, dtype=torch.int32, device=dev)


def timeit(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        f1.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


call = lambda: ctx.check(M.lib().mpsg_spmv(ctx.h, dA.h, 2, n, hx.data_ptr(), hy.data_ptr()))  # noqa
t_call = timeit(call)
t_h2d = timeit(lambda: dx.copy_(hx, non_blocking=True))
t_dev = timeit(lambda: M.spmv_dev(dA, dx.data_ptr(), dy.data_ptr(), 2, stream.cuda_stream))
t_d2h = timeit(lambda: hy.copy_(dy, non_blocking=True))
tag = os.environ.get("MPSG_PARTS", "8") + (" overlap-off" if os.environ.get("MPSG_OVERLAP") == "0" else "")
print(f"parts={tag}: call {t_call:.3f} ms ({A.nnz / t_call / 1e6:.1f} Gnnz/s) | h2d {t_h2d:.3f} dev {t_dev:.3f} "
      f"d2h {t_d2h:.3f} sum {t_h2d + t_dev + t_d2h:.3f}")
