#!/usr/bin/env python
"""PCIe copy rates for the e2e path (pinned host <-> device), 32 MB like config 2 QD x/y."""
import torch

dev = torch.device("cuda", 0)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
n = 32 * 1024 * 1024 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device=dev)
d2 = torch.empty(n, dtype=torch.float64, device=dev)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


t = timeit(lambda: d.copy_(h, non_blocking=True))
print(f"H2D 32 MB: {t * 1e3:.3f} ms = {32 * 2**20 / t / 1e9:.1f} GB/s")
t = timeit(lambda: h.copy_(d, non_blocking=True))
print(f"D2H 32 MB: {t * 1e3:.3f} ms = {32 * 2**20 / t / 1e9:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t = timeit(both)
print(f"H2D + D2H concurrent 32 MB each: {t * 1e3:.3f} ms")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max",
                      "--format=csv"], capture_output=True, text=True).stdout)
