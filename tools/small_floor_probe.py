#!/usr/bin/env python
"""Floor for a 36 MB cold-L2 kernel (config 1's SpMV moves 36 MB in one wave):
time a plain device copy of the same traffic (18 MB read + 18 MB write) and a
read-mostly reduction (32 MB read) the way kbench times a launch -- L2 flushed
before each, CUDA events around one launch, median of 30."""
import statistics

import torch

dev = torch.device("cuda", 0)
f1 = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
f2 = torch.ones(64 * 1024 * 1024, dtype=torch.int32, device=dev)


def flush():
    f1.fill_(1)
    return int(f2.sum().item() * 0)


def timed(fn, n=30):
    ts = []
    for _ in range(n):
        flush()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts), min(ts)


for mb in (4, 9, 18, 36, 72):
    n = mb * 1024 * 1024 // 8
    a = torch.rand(n, dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    med, mn = timed(lambda: b.copy_(a))
    print(f"copy {mb} MB -> {mb} MB ({2 * mb} MB traffic): median {med:.1f} us min {mn:.1f} us "
          f"({2 * mb * 1.048576 / med * 1e3:.0f} GB/s)")
    med, mn = timed(lambda: a.sum())
    print(f"sum  {mb} MB read: median {med:.1f} us min {mn:.1f} us ({mb * 1.048576 / med * 1e3:.0f} GB/s)")
med, mn = timed(lambda: None)
print(f"empty event pair: median {med:.1f} us")
