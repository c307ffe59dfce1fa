#!/usr/bin/env python
"""Short config-5 CG for profiling: python tools/cg_probe.py K iters [order]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_17510_b200 as M  # noqa: E402
import synth  # noqa: E402

K, iters = int(sys.argv[1]), int(sys.argv[2])
order = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ctx = M.Context(0)
A = synth.config_matrix(5, K)
xt = synth.config_vector(5, A.nrows, K)
dA = M.DeviceCsr(A, K, ctx=ctx)
b = M.spmv(dA, xt, M.ORDER_LANE4)
cfg = M.SolverConfig(rel_tol=1e-30, max_iters=iters, fast=order == 2, lanes_enabled=order != 0)
ts = []
for _ in range(int(os.environ.get("CG_PROBE_REPS", "3"))):
    r = M.solve_cg(M.CsrOperator(dA), b, cfg)
    ts.append(r.report.device_seconds * 1e3 / iters)
print(f"K={K} iters={r.report.iterations} device min {min(ts):.4f} median {sorted(ts)[len(ts) // 2]:.4f} ms/iter "
      f"wall {r.report.solve_seconds * 1e3 / iters:.3f} ms/iter")
