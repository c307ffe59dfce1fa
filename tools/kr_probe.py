#!/usr/bin/env python
"""Config-5 Krylov solve for A/B timing: python tools/kr_probe.py K method iters [order]
(device ms per iteration of the device-resident solve, tree dots)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_17510_b200 as M  # noqa: E402
import synth  # noqa: E402

K, method, iters = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
order = int(sys.argv[4]) if len(sys.argv) > 4 else 2
p1 = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # grid edge (0: the full config)
ctx = M.Context(0)
A = synth.config_matrix(5, K, p1=p1) if p1 else synth.config_matrix(5, K)
xt = synth.config_vector(5, A.nrows, K)
dA = M.DeviceCsr(A, K, ctx=ctx, transpose=method == "bicg")
b = M.spmv(dA, xt, M.ORDER_LANE4)
cfg = M.SolverConfig(method=M.parse_method(method), rel_tol=1e-60, max_iters=iters, fast=order == 2,
                     lanes_enabled=order != 0)
best = None
for _ in range(2):
    r = M.solve(M.CsrOperator(dA), b, cfg)
    t = r.report.device_seconds * 1e3 / max(r.report.iterations, 1)
    best = t if best is None else min(best, t)
print(f"K={K} {method} iters={r.report.iterations} {r.report.status.name} device {best:.4f} ms/iter")
