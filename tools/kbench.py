#!/usr/bin/env python
"""Kernel A/B timing helper (development tool, not the driver bench).

    MPSG_LIB=/path/variant.so python tools/kbench.py cfg2:4:2 cfg2:3:2 cfg4:2:2 ...

Each spec is cfg:K:order[:variant] (variant: pure | mixed | sptmv).  Times mpsg_spmv_dev with CUDA events on a private
stream, L2 flushed (256 MB write + 256 MB read of a second buffer) before
every timed launch, median of --steps launches; prints one line per spec.
"""
import argparse
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tag", default=os.environ.get("MPSG_LIB", "default"))
    ap.add_argument("--check", action="store_true", help="compare with the LANE4 checksum goldens")
    args = ap.parse_args()
    import torch

    import paper_2412_17510_b200 as M
    import synth

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = M.Context(0)
    ctx.set_stream(stream.cuda_stream)
    f1 = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    f2 = torch.ones(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    import ctypes

    libcuda = ctypes.CDLL("libcuda.so.1")  # demote persisting L2 lines before each flush
    cache = {}
    for spec in args.specs:
        parts = spec.split(":")
        cfg, K, order = parts[:3]
        variant = parts[3] if len(parts) > 3 else "pure"  # pure | mixed | sptmv
        c, K, order = int(cfg[3]), int(K), int(order)
        key = (c, K, variant)
        if key not in cache:
            cache.clear()
            A = synth.config_matrix(c, K)
            x = synth.config_vector(c, A.nrows, K)
            if variant == "mixed":  # the binary64 matrix: leading plane(s)
                A.planes = np.ascontiguousarray(np.stack([A.planes[0], A.planes[K]]) if c == 3 else A.planes[:1])
            cache[key] = (A, x, M.DeviceCsr(A, K, c == 3, ctx=ctx, mixed=variant == "mixed",
                                            transpose=variant == "sptmv"))
        A, x, dA = cache[key]
        n = A.nrows
        if c == 3:
            xs = [torch.from_numpy(v).to(dev) for v in x]
            ys = [torch.empty((n, K), dtype=torch.float64, device=dev) for _ in range(2)]
            if variant == "sptmv":
                step = lambda: M.sptmv_complex_dev(dA, xs[0].data_ptr(), xs[1].data_ptr(), ys[0].data_ptr(),  # noqa
                                                   ys[1].data_ptr(), order, False, stream.cuda_stream)
            else:
                step = lambda: M.spmv_complex_dev(dA, xs[0].data_ptr(), xs[1].data_ptr(), ys[0].data_ptr(),  # noqa
                                                  ys[1].data_ptr(), order, stream.cuda_stream)
        else:
            dx = torch.from_numpy(x).to(dev)
            dy = torch.empty((n, K), dtype=torch.float64, device=dev)
            if variant == "sptmv":
                step = lambda: M.sptmv_dev(dA, dx.data_ptr(), dy.data_ptr(), order, stream.cuda_stream)  # noqa
            else:
                step = lambda: M.spmv_dev(dA, dx.data_ptr(), dy.data_ptr(), order, stream.cuda_stream)  # noqa
        for _ in range(args.warmup):
            step()
        ms = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            libcuda.cuCtxResetPersistingL2Cache()
            f1.zero_()
            acc += f2.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        med = statistics.median(ms)
        extra = ""
        if args.check:
            if c == 3:
                h = M.checksum_complex(ys[0].cpu().numpy(), ys[1].cpu().numpy())
            else:
                h = M.checksum(dy.cpu().numpy())
            extra = f" checksum={h}"
        print(f"{args.tag} {spec} nnz={A.nnz} median_us={med * 1e3:.1f} min_us={min(ms) * 1e3:.1f} "
              f"gnnz_s={A.nnz / med / 1e6:.2f}{extra}", flush=True)


if __name__ == "__main__":
    main()
