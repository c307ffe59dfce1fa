#!/usr/bin/env python
"""Benchmark: multi-precision CSR SpMV / CG on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE.json configs[1] -- real QD CSR SpMV on the
random Poisson(32) matrix, n = 1,000,000 (nnz ~ 32.0M), seeded synthetic
inputs, FAST order; the TD variant of the same config is reported beside it.
One step = one y = A x over the whole matrix.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]
                    [--config cfg1..cfg5] [--K 2|3|4] [--order fast|lane4|scalar]
                    [--shard] [--cg] [--all]

Multi-GPU (torchrun, one process per GPU):
  * default (cfg2, a single-GPU config in BASELINE.json): every rank runs its
    own replica ("replicas only", weak scaling);
  * --shard (the sharded configs 3, 4, 5): the matrix is row-sharded by equal
    nnz across the ranks, x halos move over NCCL (strong scaling: value = the
    whole matrix's nnz / the max-over-ranks step time);
  * --cg (config 5): 500-iteration CG, row-sharded with --shard.

`--impl reference` times the reference's own CPU implementation (the
unmodified reference compiled from /root/reference into oracle/_ref, all host
threads) on the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "Gnnz/s for DD/TD/QD real+complex CSR SpMV; % of HBM/FP64 roofline"
CONFIG_DESC = {
    "cfg1": "2D 5-point Laplacian 512x512 (n=262144), real DD",
    "cfg2": "random Poisson(32) rows, n=1e6, real",
    "cfg3": "banded half-bandwidth 32, n=5e5, complex",
    "cfg4": "power-law Zipf(1.8) rows clipped to [1,50000], n=4e6, real DD",
    "cfg5": "3D 7-point Laplacian 128^3 (+1e-3 shift), real",
}
# fp64 operations per nonzero for one mul + one add in the reference op
# sequence (counted with the reference's templated chains)
OPS_PER_NNZ = {2: 20, 3: 202, 4: 206}
# Mixed mode (binary64 matrix): one mul_by_double + one add
OPS_PER_NNZ_MIXED = {2: 17, 3: 130, 4: 152}
# FAST order executes a fused product-accumulate (mc_arith.cuh fma_acc /
# fma_fast): the running accumulator is updated level by level (QD: 6
# two_prods 12 + 14 two_sums 84 + level-3 sum 16 + sweep 9 = 121; TD: 6 + 5
# two_sums 30 + level-2 sum 10 + sweep 6 = 52; DD: 6 + 11 = 17), one
# canonicalising renorm per row (QD 22, TD 16), and
# stored vector updates = the accumulate + the full renorm (QD 143, TD 68).  The roofline of
# a FAST line counts the operations it executes; the reference's count and the
# fraction against it are reported beside (reference_fp64_ops, reference_frac).
OPS_FAST = {2: 17, 3: 52, 4: 121}
OPS_FAST_MIXED = {2: 17, 3: 114, 4: 76}
OPS_FAST_UPDATE = {2: 20, 3: 68, 4: 143}
# Real short rows (sell_real_kernel, FAST): the products of a round of G go
# into unnormalised level sums (fma_lvl: QD 12 + 84 + 16 = 112, TD 6 + 30 + 9 =
# 45; Mixed QD 67, TD 33) and the backward sweep (QD 9, TD 6) runs once per
# round (G = 4 QD, 2 TD), once more at the row's end, then the row's renorm.
OPS_FAST_SELL = {2: 17, 3: 45 + 6 / 2, 4: 112 + 9 / 4}
OPS_FAST_SELL_MIXED = {2: 17, 3: 33 + 6 / 2, 4: 67 + 9 / 4}
ROW_CANON = {2: 0, 3: 16 + 6, 4: 22 + 9}
K_NAME = {2: "DD", 3: "TD", 4: "QD"}
ORDER_NAME = {0: "scalar", 1: "lane4", 2: "fast"}
CG_ITERS = 500


def algorithmic_bytes(nnz, n, K, cplx, mixed=False):
    c = 2 if cplx else 1
    # matrix planes (K, or 1 binary64 plane in mixed mode) + int32 columns +
    # int32 row pointer + x read once + y written once
    return nnz * (8 * (1 if mixed else K) * c + 4) + 4 * (n + 1) + 2 * n * 8 * K * c


def algorithmic_ops(nnz, K, cplx, mixed=False, n=0, fast=False):
    if fast and cplx:  # four real sums per nonzero; Pure keeps the sweep per product (fma_acc)
        return nnz * 4 * (OPS_FAST_SELL_MIXED if mixed else OPS_FAST)[K]
    if fast:
        per = (OPS_FAST_SELL_MIXED if mixed else OPS_FAST_SELL)[K]
        return nnz * per + n * ROW_CANON[K]
    return nnz * (OPS_PER_NNZ_MIXED if mixed else OPS_PER_NNZ)[K] * (4 if cplx else 1)


def cg_iter_bytes(nnz, n, K):
    # SpMV + x, r, p read/write + q write/read
    return nnz * (8 * K + 4) + 4 * (n + 1) + 11 * n * 8 * K


def cg_iter_ops(nnz, n, K, fast=False):
    if fast:  # SpMV + <p,q>, <r,r> accumulations + x, r, p stored updates (cg_kernels.cuh)
        vec = 2 * OPS_FAST[K] + 3 * OPS_FAST_UPDATE[K] if K > 2 else 5 * OPS_PER_NNZ[K]
        return nnz * OPS_FAST_SELL[K] + n * ROW_CANON[K] + n * vec
    return (nnz + 5 * n) * OPS_PER_NNZ[K]


# Per-iteration algorithmic work of the other device solvers (krylov_inst.cuh),
# as (SpMVs, multi-component mul+add pairs per element, vector passes of n*8K
# bytes incl. each SpMV's input and output):
#   BiCGSTAB: <r~,v>; s = r - alpha v, <s,s>; <t,t>, <t,s>; x += alpha p + omega s,
#   r = s - omega t, <r,r>, <r~,r>; p = r + beta (p - omega v)  -> 2 SpMV, 12 pairs, 22 passes
SOLVER_WORK = {"bicgstab": (2, 12, 22)}
SOLVER_ITERS = 200


def solver_iter_bytes(method, nnz, n, K):
    s, _, passes = SOLVER_WORK[method]
    return s * (nnz * (8 * K + 4) + 4 * (n + 1)) + passes * n * 8 * K


def solver_iter_ops(method, nnz, n, K, fast=False):
    s, pairs, _ = SOLVER_WORK[method]
    if fast:  # BiCGSTAB: 6 dot accumulations, 5 fused stored updates, 1 plain (p - omega v)
        vec = 6 * OPS_FAST[K] + 5 * OPS_FAST_UPDATE[K] + OPS_PER_NNZ[K] if K > 2 else pairs * OPS_PER_NNZ[K]
        return s * (nnz * OPS_FAST_SELL[K] + n * ROW_CANON[K]) + n * vec
    return (s * nnz + pairs * n) * OPS_PER_NNZ[K]


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json (copy kernel)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_for(key):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(key)
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx = float(s[1])
                for nm, v in zip(names, s[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(cfg: str, K: int, mixed: bool = False):
    c = int(cfg[3])
    A = synth.config_matrix(c, K)
    x = synth.config_vector(c, A.nrows, K)
    if mixed:  # the binary64 matrix of Mixed mode: the leading value plane(s)
        A.planes = np.ascontiguousarray(np.stack([A.planes[0], A.planes[K]]) if c == 3 else A.planes[:1])
    return A, x


# --------------------------------------------------------------------------- reference arm
def run_reference(steps, warmup, cfg, K, cg=False, threads=None, order=1, inputs=None):
    """Time the unmodified reference (oracle/_ref: mps::spmv / mps::solve_cg) on host cores.
    order 1 = lanes on, the reference default (kernels.hpp:44)."""
    import oracle as O

    threads = threads or os.cpu_count() or 1
    A, x = inputs or make_inputs(cfg, K)
    cplx = cfg == "cfg3"
    kind = "reference" if O.ref_available() else "port"
    nnz = A.nnz
    if isinstance(cg, str) and cg != "cg":
        # a bounded prefix of the solve (serial vector ops, krylov.hpp:122-140)
        iters = 2
        if kind == "reference":
            b = O.ref_spmv(A, x, order, threads=threads)
            call = lambda: O.ref_solve(A, b, cg, order, threads=threads, rel_tol=1e-99, max_iters=iters)  # noqa
        else:
            threads = 1
            b = O.spmv(A, x, order)
            call = lambda: O.solve(A, b, cg, order, rel_tol=1e-99, max_iters=iters)  # noqa: E731
        units = SOLVER_WORK[cg][0] * nnz * iters
        sample = (f"cfg5 {K_NAME[K]} {cg}, first {iters} of {SOLVER_ITERS} iterations (SpMV on {threads} "
                  f"OpenMP threads, vector ops serial as in krylov.hpp:122-140)")
    elif cg:
        # a bounded prefix of the 500-iteration solve (the serial vector ops of
        # krylov.hpp:122-140 dominate; the full run is minutes to tens of minutes)
        iters = 3
        if kind == "reference":
            b = O.ref_spmv(A, x, order, threads=threads)
            call = lambda: O.ref_cg(A, b, order, threads=threads, rel_tol=1e-30, max_iters=iters)  # noqa: E731
        else:
            threads = 1
            b = O.spmv(A, x, order)
            call = lambda: O.cg(A, b, order, rel_tol=1e-30, max_iters=iters)  # noqa: E731
        units = nnz * iters
        sample = (f"cfg5 {K_NAME[K]} CG, first {iters} of {CG_ITERS} iterations (SpMV on {threads} OpenMP "
                  f"threads, vector ops serial as in krylov.hpp:122-140)")
    else:
        if kind == "reference":
            if cplx:
                Ah, xh, yh = O.RefComplex(A, K), O.RefCVec(*x), O.RefCVec(K=K)
                call = lambda: O.ref().ref_spmv_complex(Ah.h, xh.h, order, threads, yh.h)  # noqa: E731
            else:
                Ah, xh, yh = O.RefCsr(A, K), O.RefVec(x), O.RefVec(K=K)
                call = lambda: O.ref().ref_spmv(Ah.h, xh.h, order, threads, yh.h)  # noqa: E731
        else:
            threads = 1
            call = (lambda: O.spmv_complex(A, x[0], x[1], order)) if cplx else (lambda: O.spmv(A, x, order))
        units = nnz
        sample = (f"{cfg} {K_NAME[K]} {'complex ' if cplx else ''}full matrix (nnz={nnz}), "
                  f"lanes {'on' if order == 1 else 'off'}, {threads} OpenMP threads")
    for _ in range(warmup):
        call()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return dict(value=units / med / 1e9, median_s=med, cores=threads, kind=kind,
                sample=sample + f", median of {len(times)} timed calls after {warmup} warm-up")


# --------------------------------------------------------------------------- GPU arm
class Flush:
    """L2 flush before a timed step: write a 256 MB buffer (> 126 MB L2), then
    read a second 256 MB buffer so the write's dirty lines are evicted before
    the timed launch (the kernel starts with a cold, clean L2)."""

    def __init__(self, torch, dev):
        self.w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
        self.r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
        self.acc = torch.zeros(1, dtype=torch.int64, device=dev)

    def __call__(self):
        self.w.zero_()
        self.acc.add_(self.r.sum())


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            return next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), "unknown")
    except OSError:
        return "unknown"


def best_reference(steps, warmup, cfg, K, light=False):
    """The fastest way the reference computes this SpMV on this host: lanes on
    (its default) and off, its own flags and the x86-64-v3 build (all
    bit-identical), every host thread.  Each combination is screened with
    1 warm-up + 2 timed calls; the fastest is then timed with steps / warmup.
    Returns (result, rows) where rows holds every screened combination plus
    one thread, for SURVEY 8(d)'s CPU table."""
    import oracle as O

    inputs = make_inputs(cfg, K)
    if not O.ref_available():
        return run_reference(steps, warmup, cfg, K, inputs=inputs), None
    rows, best = {}, None
    builds = [False] + ([True] if O.use_ref_build(True) and O.use_ref_build(False) else [])
    for v3 in builds:
        O.use_ref_build(v3)
        try:
            for order in (1, 0):
                r = run_reference(1 if light else 2, 1, cfg, K, order=order, inputs=inputs)
                label = f"{'x86-64-v3 build' if v3 else 'reference flags'}, lanes {'on' if order else 'off'}, " \
                        f"threads={r['cores']}"
                rows[label] = r["value"]
                if best is None or r["value"] > best[0]:
                    best = (r["value"], v3, order, label)
        finally:
            O.use_ref_build(False)
    rows["reference flags, lanes on, threads=1"] = run_reference(1 if light else 2, 0 if light else 1, cfg, K,
                                                                 threads=1, inputs=inputs)["value"]
    _, v3, order, label = best
    O.use_ref_build(v3)
    try:
        r = run_reference(steps, warmup, cfg, K, order=order, inputs=inputs)
    finally:
        O.use_ref_build(False)
    r["sample"] = f"{r['sample']} [fastest reference variant: {label}]"
    return r, {"unit": "Gnnz/s", "rows": rows, "chosen": label, "cpu": cpu_model(), "nproc": os.cpu_count()}


def setup_stream(torch, M, dev):
    # a dedicated (non-default) stream: every launch of ours and every timing
    # event goes on it (torch's legacy default stream has handle 0, which the C
    # ABI reads as "the context's own stream")
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = M.Context(dev.index)
    ctx.set_stream(stream.cuda_stream)
    return stream, ctx


def make_comm(M, ctx, world, rank, dist):
    uid = [M.Comm.unique_id() if (rank == 0 and world > 1) else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    return M.Comm(ctx, world, rank, uid[0])


def max_over_ranks(torch, dev, dist, v):
    if not dist:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_gpu_spmv(args, cfg, K, order, rank, world, dist, variant="pure"):
    """variant: "pure" (A in K components), "mixed" (binary64 A), "sptmv" (y = A^T x)."""
    import torch

    import paper_2412_17510_b200 as M

    dev = torch.device("cuda", torch.cuda.current_device())
    stream, ctx = setup_stream(torch, M, dev)
    cplx = cfg == "cfg3"
    mixed, trans = variant == "mixed", variant == "sptmv"
    A, x = make_inputs(cfg, K, mixed)
    n, nnz = A.nrows, A.nnz
    shard = args.shard and world > 1 and variant == "pure"
    xs = list(x) if cplx else [x]
    comm = None
    if shard:
        comm = make_comm(M, ctx, world, rank, dist)
        dA = M.DistCsr.from_global(comm, A, K, cplx)
        b, e = dA.row_begin, dA.row_end
        _, halo = dA.info()
        dxs = [torch.from_numpy(np.ascontiguousarray(v[b:e])).to(dev) for v in xs]
        dys = [torch.empty((e - b, K), dtype=torch.float64, device=dev) for _ in xs]
        if cplx:
            step = lambda: M.dspmv_complex_dev(dA, dxs[0].data_ptr(), dxs[1].data_ptr(), dys[0].data_ptr(),  # noqa
                                               dys[1].data_ptr(), order, stream.cuda_stream)
        else:
            step = lambda: M.dspmv_dev(dA, dxs[0].data_ptr(), dys[0].data_ptr(), order, stream.cuda_stream)  # noqa
        local_stats = None
        units = nnz  # strong scaling: the whole matrix per step across the group
    else:
        dA = M.DeviceCsr(A, K, cplx, ctx=ctx, mixed=mixed, transpose=trans)
        local_stats = dA.stats()
        halo = 0
        dxs = [torch.from_numpy(v).to(dev) for v in xs]
        dys = [torch.empty((n, K), dtype=torch.float64, device=dev) for _ in xs]
        if trans and cplx:
            step = lambda: M.sptmv_complex_dev(dA, dxs[0].data_ptr(), dxs[1].data_ptr(), dys[0].data_ptr(),  # noqa
                                               dys[1].data_ptr(), order, False, stream.cuda_stream)
        elif trans:
            step = lambda: M.sptmv_dev(dA, dxs[0].data_ptr(), dys[0].data_ptr(), order, stream.cuda_stream)  # noqa
        elif cplx:
            step = lambda: M.spmv_complex_dev(dA, dxs[0].data_ptr(), dxs[1].data_ptr(), dys[0].data_ptr(),  # noqa
                                              dys[1].data_ptr(), order, stream.cuda_stream)
        else:
            step = lambda: M.spmv_dev(dA, dxs[0].data_ptr(), dys[0].data_ptr(), order, stream.cuda_stream)  # noqa
        units = world * nnz  # replicas (weak scaling)
    flush = Flush(torch, dev)
    for _ in range(args.warmup):
        flush()
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clk = ClockSampler(dev.index)
    clk.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush()
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = clk.stop()
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_total = max_over_ranks(torch, dev, dist, sum(ms) / 1e3)

    # e2e through the host-pointer C-ABI call (pinned host buffers, H2D + D2H inside)
    e2e = e2e_pageable = None
    if not args.no_e2e and not shard and variant == "pure":
        if cplx:
            hx = [torch.from_numpy(v).pin_memory() for v in xs]
            hy = [torch.empty((n, K), dtype=torch.float64).pin_memory() for _ in range(2)]
            call = lambda: M.lib().mpsg_spmv_complex(ctx.h, dA.h, order, n, hx[0].data_ptr(), hx[1].data_ptr(),  # noqa
                                                     hy[0].data_ptr(), hy[1].data_ptr())
            h2d, d2h = 2 * n * K * 8, 2 * n * K * 8
        else:
            hx = torch.from_numpy(x).pin_memory()
            hy = torch.empty((n, K), dtype=torch.float64).pin_memory()
            call = lambda: M.lib().mpsg_spmv(ctx.h, dA.h, order, n, hx.data_ptr(), hy.data_ptr())  # noqa: E731
            h2d, d2h = n * K * 8, n * K * 8
        for _ in range(max(1, args.warmup)):
            flush()
            ctx.check(call())
        ets = []
        if dist:
            dist.barrier()
        for _ in range(args.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.check(call())
            e1.record(stream)
            torch.cuda.synchronize()
            ets.append(e0.elapsed_time(e1) / 1e3)
        te = max_over_ranks(torch, dev, dist, sum(ets))
        e2e = {"value": world * nnz * args.steps / te / 1e9, "unit": "Gnnz/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "call": "mpsg_spmv_complex" if cplx else "mpsg_spmv",
               "host_memory": "pinned"}
        # the same call on pageable host arrays (numpy, like the drop-in's
        # std::vector): the library stages them through its own pinned chunks
        if cplx:
            px = [np.ascontiguousarray(v) for v in xs]
            py = [np.empty((n, K)) for _ in range(2)]
            pcall = lambda: M.lib().mpsg_spmv_complex(ctx.h, dA.h, order, n, px[0].ctypes.data, px[1].ctypes.data,  # noqa
                                                      py[0].ctypes.data, py[1].ctypes.data)
        else:
            px, py = np.ascontiguousarray(x), np.empty((n, K))
            pcall = lambda: M.lib().mpsg_spmv(ctx.h, dA.h, order, n, px.ctypes.data, py.ctypes.data)  # noqa: E731
        ctx.check(pcall())
        pts = []
        for _ in range(args.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.check(pcall())
            e1.record(stream)
            torch.cuda.synchronize()
            pts.append(e0.elapsed_time(e1) / 1e3)
        tp = max_over_ranks(torch, dev, dist, sum(pts))
        e2e_pageable = {"value": world * nnz * args.steps / tp / 1e9, "unit": "Gnnz/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "call": e2e["call"], "host_memory": "pageable (numpy)"}
    if local_stats is not None:
        kernels = (1 if local_stats.nslices > 0 else 0) + (1 if local_stats.nlong > 0 else 0)
        # real TD, FAST order, dense-enough matrices: x is first re-laid out to 32 bytes per element (pad_td_kernel)
        if (K == 3 and not cplx and not mixed and order == 2 and nnz >= (1 << 20)
                and nnz - local_stats.long_nnz >= 12 * local_stats.ncols):
            kernels += 1
    else:
        kernels = 2  # upper bound for a shard (SELL + long-row kernel)
    # a working set that fits in L2 (config 1: 36 MB of 126 MB) also reported
    # L2-warm: back-to-back launches, no flush (SURVEY 8(d) timing protocol)
    l2_warm = None
    if not shard and algorithmic_bytes(nnz, n, K, cplx, mixed) < 64e6:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        step()
        e0.record(stream)
        for _ in range(reps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        tw = e0.elapsed_time(e1) / 1e3 / reps
        l2_warm = {"value": nnz / tw / 1e9, "unit": "Gnnz/s", "us_per_step": tw * 1e6,
                   "note": f"{reps} back-to-back launches, L2 not flushed (working set fits in L2)"}
    res = dict(n=n, nnz=nnz, units=units, t_total=t_total, per_launch=t_total / args.steps, clocks=clocks,
               e2e=e2e, e2e_pageable=e2e_pageable, launches=args.steps * kernels, cplx=cplx, halo_rows=halo,
               shard=shard, variant=variant, l2_warm=l2_warm, order=order)
    del dA
    if comm:
        comm.close()
    ctx.close()
    return res


def run_gpu_cg(args, K, order, rank, world, dist, method="cg"):
    """Config 5: 500 CG iterations (fixed budget, rel_tol 1e-30 so none stops early);
    method != "cg": that device solver (mpsg_solve, tree dots) for up to
    SOLVER_ITERS iterations, units = SpMVs x nnz x iterations done."""
    import torch

    import paper_2412_17510_b200 as M

    dev = torch.device("cuda", torch.cuda.current_device())
    stream, ctx = setup_stream(torch, M, dev)
    A, xt = make_inputs("cfg5", K)
    n, nnz = A.nrows, A.nnz
    shard = args.shard and world > 1 and method == "cg"
    iters = CG_ITERS if method == "cg" else SOLVER_ITERS
    cfg = M.SolverConfig(method=M.parse_method(method), rel_tol=1e-30 if method == "cg" else 1e-99,
                         max_iters=iters, lanes_enabled=order != 0, fast=order == 2,
                         cg_variant=getattr(args, "cg_variant", 0))
    comm = None
    if method != "cg":
        dA = M.DeviceCsr(A, K, ctx=ctx)
        b = M.spmv(dA, xt, M.ORDER_LANE4)
        op = M.CsrOperator(dA)
        solve = lambda: M.solve(op, b, cfg)  # noqa: E731
        units = None
    elif shard:
        comm = make_comm(M, ctx, world, rank, dist)
        dA = M.DistCsr.from_global(comm, A, K)
        b0, e0 = dA.row_begin, dA.row_end
        bfull = M.spmv(M.DeviceCsr(A, K, ctx=ctx), xt, M.ORDER_LANE4)
        b = np.ascontiguousarray(bfull[b0:e0])
        solve = lambda: M.dsolve_cg(dA, b, cfg)  # noqa: E731
        units = nnz * CG_ITERS
    else:
        dA = M.DeviceCsr(A, K, ctx=ctx)
        b = M.spmv(dA, xt, M.ORDER_LANE4)
        op = M.CsrOperator(dA)
        solve = lambda: M.solve_cg(op, b, cfg)  # noqa: E731
        units = world * nnz * CG_ITERS
    for _ in range(max(1, args.warmup // 3)):
        solve()
    clk = ClockSampler(dev.index)
    clk.start()
    if dist:
        dist.barrier()
    loop, wall, res = [], [], None
    for _ in range(max(3, args.steps // 5)):  # whole solves; medians below
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = solve()
        wall.append(time.perf_counter() - t0)
        loop.append(res.report.device_seconds)
    if dist:
        dist.barrier()
    clocks = clk.stop()
    t_loop = max_over_ranks(torch, dev, dist, statistics.median(loop))
    t_wall = max_over_ranks(torch, dev, dist, statistics.median(wall))
    rep = res.report
    if units is None:  # other solvers: the iterations actually run
        iters = max(rep.iterations, 1)
        units = world * SOLVER_WORK[method][0] * nnz * iters
    out = dict(n=n, nnz=nnz, units=units, t_total=t_loop, per_iter=t_loop / iters, clocks=clocks,
               e2e={"value": units / t_wall / 1e9, "unit": f"Gnnz/s ({method} SpMV work)",
                    "h2d_bytes_per_step": int(b.nbytes), "d2h_bytes_per_step": int(b.nbytes) + 8 * (iters + 1),
                    "call": "mpsg_dcg" if shard else ("mpsg_cg" if method == "cg" else "mpsg_solve")},
               method=method, iters=iters,
               iterations=rep.iterations, rel_residual=rep.residual_history[-1] / rep.residual_history[0],
               true_residual=rep.final_true_residual, shard=shard, cplx=False, halo_rows=0,
               launches=iters * (5 if method == "cg" else 9))
    del dA
    if comm:
        comm.close()
    ctx.close()
    return out


def roofline(kind, nnz, n, K, cplx, seconds, hbm_peak, fp64_peak, tkey, mixed=False, fast=False):
    if kind == "cg":
        byts = cg_iter_bytes(nnz, n, K)
        ops, ref_ops = cg_iter_ops(nnz, n, K, fast), cg_iter_ops(nnz, n, K)
    elif kind in SOLVER_WORK:
        byts = solver_iter_bytes(kind, nnz, n, K)
        ops, ref_ops = solver_iter_ops(kind, nnz, n, K, fast), solver_iter_ops(kind, nnz, n, K)
    else:
        byts = algorithmic_bytes(nnz, n, K, cplx, mixed)
        ops, ref_ops = algorithmic_ops(nnz, K, cplx, mixed, n, fast), algorithmic_ops(nnz, K, cplx, mixed)
    t_hbm, t_fp = byts / (hbm_peak * 1e9), ops / fp64_peak
    if t_hbm >= t_fp:
        ach = byts / seconds / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    else:
        ach = ops / seconds / 1e12
        pk = fp64_peak / 1e12
        roof = {"bound": "fp64", "achieved": ach, "peak": pk, "unit": "T fp64 instr/s", "frac": ach / pk,
                "peak_source": "measured on this GPU by mpsg_measure_fp64_peak (DFMA throughput)"}
        if ops != ref_ops:  # FAST: executed fused arithmetic; the reference algorithm's count beside
            roof.update(reference_fp64_ops=ref_ops, reference_frac=ref_ops / seconds / fp64_peak,
                        ops_note="fp64 ops of the executed FAST arithmetic (fused product-accumulate, "
                                 "bench.py OPS_FAST); reference_frac counts the reference algorithm's ops")
    roof.update(t_roofline_us=max(t_hbm, t_fp) * 1e6, algorithmic_bytes=byts, algorithmic_fp64_ops=ops,
                per=(f"one {kind} iteration" if kind != "spmv" else "one SpMV launch"),
                traffic=traffic_for(tkey))
    return roof


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--K", type=int, default=4)
    ap.add_argument("--order", default="fast", choices=["fast", "lane4", "scalar"])
    ap.add_argument("--shard", action="store_true", help="row-shard the matrix across ranks (configs 3, 4, 5)")
    ap.add_argument("--cg", action="store_true", help="config 5: 500-iteration CG instead of one SpMV")
    ap.add_argument("--cg-variant", type=int, default=0, choices=[0, 1, 2],
                    help="--cg: 0 auto (classic on one GPU, one reduction per iteration when sharded), 1 classic, 2 one reduction")
    ap.add_argument("--solver", default="", help="config 5: a device solver (bicgstab) instead of one SpMV")
    ap.add_argument("--variant", default="pure", choices=["pure", "mixed", "sptmv"],
                    help="mixed: binary64 matrix (the paper's M mode); sptmv: y = A^T x")
    ap.add_argument("--all", action="store_true", help="one line per config/precision (not the driver line)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--secondary", default="", help="'none' disables the TD line beside the cfg2 QD headline")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.solver == "cg":
        args.cg, args.solver = True, ""
    if args.cg or args.solver:
        args.config = "cfg5"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    order = {"fast": 2, "lane4": 1, "scalar": 0}[args.order]

    if args.impl == "reference":
        if rank != 0:
            return 0
        variants = None
        if args.cg or args.solver:
            r = run_reference(args.steps, args.warmup, args.config, args.K, cg=args.solver or args.cg)
        else:
            r, variants = best_reference(args.steps, args.warmup, args.config, args.K)
        line = {"metric": METRIC, "value": r["value"], "unit": "Gnnz/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["median_s"] * 1e3, "higher_is_better": True,
                "scaling": "strong" if args.shard else "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generators, synth/mpsgen.c)", "impl": "reference",
                "config": {"workload": f"{args.config} {K_NAME[args.K]}"
                                       f"{(' ' + (args.solver or 'cg').upper()) if (args.cg or args.solver) else ''}: "
                                       f"{CONFIG_DESC[args.config]}",
                           "precision": K_NAME[args.K],
                           "order": variants["chosen"] if variants else "lane4 (reference default)"},
                "cpu_baseline": {"value": r["value"], "unit": "Gnnz/s", "cores": r["cores"], "kind": r["kind"],
                                 "sample": r["sample"]},
                "e2e": {"value": r["value"], "unit": "Gnnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        if variants:
            line["cpu_variants"] = variants
        print(json.dumps(line), flush=True)
        return 0

    import torch

    dist = None
    if world > 1:
        import torch.distributed as tdist

        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
    else:
        torch.cuda.set_device(0)

    import paper_2412_17510_b200 as M

    hbm_peak, _ = measured_peaks()
    probe = M.Context(torch.cuda.current_device())
    fp64_peak = M.measure_fp64_peak(probe)
    probe.close()

    jobs = [(args.config, args.K, args.solver or args.cg, args.variant, order)]
    if args.all:
        spmv = [("cfg1", 2), ("cfg2", 3), ("cfg2", 4), ("cfg3", 2), ("cfg3", 4), ("cfg4", 2), ("cfg5", 2), ("cfg5", 4)]
        jobs = [(c, k, False, "pure", order) for c, k in spmv]
        jobs += [("cfg5", 2, True, "pure", order), ("cfg5", 4, True, "pure", order),
                 ("cfg2", 4, False, "mixed", order), ("cfg4", 2, False, "mixed", order),
                 ("cfg3", 4, False, "mixed", order), ("cfg2", 4, False, "sptmv", order),
                 ("cfg3", 2, False, "sptmv", order), ("cfg5", 2, "bicgstab", "pure", order),
                 ("cfg5", 4, "bicgstab", "pure", order)]
        if order != 1:  # the bit-exact LANE4 order (the reference default, kernels.hpp:44) per SpMV config
            jobs += [(c, k, False, "pure", 1) for c, k in spmv]
    secondary = None
    if (not args.all and args.config == "cfg2" and args.K == 4 and not args.cg and args.variant == "pure"
            and args.secondary != "none"):
        secondary = ("cfg2", 3, False, "pure", order)

    results = []
    for cfg, K, cg, variant, jorder in jobs + ([secondary] if secondary else []):
        if cg:
            meth = cg if isinstance(cg, str) else "cg"
            r = run_gpu_cg(args, K, jorder, rank, world, dist, meth)
            r["variant"] = "pure"
            r["order"] = jorder
            r["roof"] = roofline(meth, r["nnz"], r["n"], K, False, r["per_iter"], hbm_peak, fp64_peak,
                                 f"cg5_K{K}" if meth == "cg" else f"{meth}5_K{K}", fast=jorder == 2)
        else:
            r = run_gpu_spmv(args, cfg, K, jorder, rank, world, dist, variant)
            tkey = f"{cfg}_K{K}" + ("" if variant == "pure" else f"_{variant}") + ("" if jorder == 2 else f"_o{jorder}")
            r["roof"] = roofline("spmv", r["nnz"], r["n"], K, r["cplx"], r["per_launch"], hbm_peak, fp64_peak,
                                 tkey, mixed=variant == "mixed", fast=jorder == 2)
        results.append((cfg, K, cg, r))

    cpu_cache = {}
    if rank == 0:
        for idx, (cfg, K, cg, r) in enumerate(results[: len(jobs)]):
            vname = {"pure": "", "mixed": " Mixed (binary64 matrix)", "sptmv": " SpTMV y=A^T x"}[r["variant"]]
            steps = 1 if cg else args.steps
            value = r["units"] * steps / r["t_total"] / 1e9
            if r["shard"]:
                par = f"row-sharded x{world} (equal-nnz blocks, NCCL x halo)"
            else:
                par = f"replicas x{world}" if world > 1 else "single GPU"
            line = {"metric": METRIC, "value": value, "unit": "Gnnz/s", "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup,
                    "ms_per_step": (r["t_total"] * 1e3 if cg else r["t_total"] / args.steps * 1e3),
                    "higher_is_better": True, "scaling": "strong" if r["shard"] else "weak",
                    "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic (seeded generators, synth/mpsgen.c)",
                    "config": {"workload": f"{cfg} {K_NAME[K]}"
                                           f"{(' ' + r['method'].upper() + ' x' + str(r['iters'])) if cg else ''}"
                                           f"{vname}: {CONFIG_DESC[cfg]}",
                               "precision": K_NAME[K], "order": ORDER_NAME[r["order"]], "nnz": r["nnz"],
                               "n": r["n"],
                               "parallelism": par,
                               "l2": ("flushed before every timed step: 256 MB write, then 256 MB read of a "
                                      "second buffer") if not cg else "inputs (A, vectors) larger than L2"},
                    "roofline": r["roof"], "clocks": r["clocks"], "e2e": r["e2e"], "gpu_launches": r["launches"]}
            if r.get("e2e_pageable"):
                line["e2e_pageable"] = r["e2e_pageable"]
            if cg:
                line["config"].update(step=f"one {r['iters']}-iteration {r['method']} solve (graph-captured "
                                           "batches of 32)",
                                      iterations=r["iterations"], rel_residual=r["rel_residual"],
                                      true_residual=r["true_residual"])
                if r["method"] == "cg":
                    one = args.cg_variant == 2 or (args.cg_variant == 0 and r["shard"])
                    line["config"]["cg_form"] = ("one reduction per iteration (Chronopoulos-Gear)" if one else
                                                 "reference form, two reductions per iteration")
                line["ms_per_iteration"] = r["per_iter"] * 1e3
            if r["shard"]:
                line["config"]["halo_rows_rank0"] = r["halo_rows"]
            if r.get("l2_warm"):
                line["l2_warm"] = r["l2_warm"]
            if secondary and idx == 0:
                c2, k2, _, r2 = results[-1]
                line["secondary"] = {"workload": f"{c2} {K_NAME[k2]}",
                                     "value": r2["units"] * args.steps / r2["t_total"] / 1e9,
                                     "unit": "Gnnz/s", "roofline": r2["roof"], "e2e": r2["e2e"]}
            if world == 1 and not args.no_cpu and r["variant"] == "pure" and (not args.all or not cg):
                key = (cfg, K, cg)
                if key not in cpu_cache:
                    if cg:
                        cpu_cache[key] = (run_reference(1, 0, cfg, K, cg=cg), None)
                    else:  # --all: a lighter screen (1 timed call per variant) keeps the run to minutes
                        cpu_cache[key] = best_reference(2 if args.all else 5, 1, cfg, K, light=args.all)
                cb, cvar = cpu_cache[key]
                if cvar:
                    line["cpu_variants"] = cvar
                line["cpu_baseline"] = {"value": cb["value"], "unit": "Gnnz/s", "cores": cb["cores"],
                                        "kind": cb["kind"], "sample": cb["sample"]}
                if cvar and "reference flags, lanes on, threads=1" in cvar["rows"]:
                    line["cpu_baseline"]["one_thread"] = cvar["rows"]["reference flags, lanes on, threads=1"]
            print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
