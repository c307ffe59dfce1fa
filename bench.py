#!/usr/bin/env python
"""Benchmark: multi-precision CSR SpMV on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE.json configs[1] -- real QD CSR SpMV on the
random Poisson(32) matrix, n = 1,000,000 (nnz ~ 32.0M), seeded synthetic
inputs; the TD variant of the same config is reported beside it.  One step =
one y = A x over the whole matrix.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]
                    [--config cfg2] [--K 4] [--order fast|lane4|scalar] [--all]

Under torchrun (N > 1) every rank runs its own replica of the single-GPU
config (configs[1] does not shard: "replicas only", weak scaling); timing is
the max over ranks of the device-timed region.

`--impl reference` times the reference's own CPU implementation (the
unmodified reference compiled from /root/reference into oracle/_ref, run with
all host threads) on the same config; rank 0 only.
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
K_NAME = {2: "DD", 3: "TD", 4: "QD"}


def algorithmic_bytes(nnz, n, K, cplx):
    c = 2 if cplx else 1
    # matrix planes + int32 columns + int32 row pointer + x read once + y written once
    return nnz * (8 * K * c + 4) + 4 * (n + 1) + 2 * n * 8 * K * c


def algorithmic_ops(nnz, K, cplx):
    return nnz * OPS_PER_NNZ[K] * (4 if cplx else 1)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json"
    return 6650.0, "fallback (B200_PROFILING.md)"


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


def make_inputs(cfg: str, K: int):
    c = int(cfg[3])
    A = synth.config_matrix(c, K)
    x = synth.config_vector(c, A.nrows, K)
    return A, x


# --------------------------------------------------------------------------- reference arm
def run_reference(args, cfg, K, sample_rows=None):
    """Time the unmodified reference spmv (oracle/_ref) on host cores."""
    import oracle as O

    threads = os.cpu_count() or 1
    A, x = make_inputs(cfg, K)
    cplx = cfg == "cfg3"
    kind = "reference" if O.ref_available() else "port"
    if sample_rows and sample_rows < A.nrows:
        from types import SimpleNamespace

        nnz_s = int(A.indptr[sample_rows])
        A = SimpleNamespace(nrows=sample_rows, ncols=A.ncols, indptr=A.indptr[: sample_rows + 1],
                            indices=A.indices[:nnz_s], planes=A.planes[:, :nnz_s], K=K, nnz=nnz_s)
    nnz = int(A.indptr[A.nrows])
    order = 1  # lanes on: the reference default (kernels.hpp:44)
    times = []
    if kind == "reference":
        if cplx:
            Ah, xh, yh = O.RefComplex(A, K), O.RefCVec(*x), O.RefCVec(K=K)
            call = lambda: O.ref().ref_spmv_complex(Ah.h, xh.h, order, threads, yh.h)  # noqa: E731
        else:
            Ah, xh, yh = O.RefCsr(A, K), O.RefVec(x), O.RefVec(K=K)
            call = lambda: O.ref().ref_spmv(Ah.h, xh.h, order, threads, yh.h)  # noqa: E731
        threads_used = threads
    else:
        call = (lambda: O.spmv_complex(A, x[0], x[1], order)) if cplx else (lambda: O.spmv(A, x, order))
        threads_used = 1
    for _ in range(args.warmup):
        call()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return dict(value=nnz / med / 1e9, seconds=sum(times), median_s=med, cores=threads_used, kind=kind,
                sample=(f"{cfg} {K_NAME[K]} {'complex ' if cplx else ''}rows [0,{A.nrows}) nnz={nnz}, "
                        f"lanes on, {threads_used} OpenMP threads, median of {len(times)} calls"))


# --------------------------------------------------------------------------- GPU arm
def run_gpu(args, cfg, K, order, rank, world, dist):
    import torch

    import paper_2412_17510_b200 as M

    dev = torch.device("cuda", torch.cuda.current_device())
    # a dedicated (non-default) stream: every launch of ours and every timing
    # event goes on it (torch's legacy default stream has handle 0, which the
    # C ABI reads as "the context's own stream")
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = M.Context(dev.index)
    ctx.set_stream(stream.cuda_stream)
    cplx = cfg == "cfg3"
    A, x = make_inputs(cfg, K)
    dA = M.DeviceCsr(A, K, cplx, ctx=ctx)
    st = dA.stats()
    n, nnz = A.nrows, A.nnz
    if cplx:
        dxr, dxi = torch.from_numpy(x[0]).to(dev), torch.from_numpy(x[1]).to(dev)
        dyr, dyi = torch.empty((n, K), dtype=torch.float64, device=dev), torch.empty((n, K), dtype=torch.float64,
                                                                                     device=dev)
        step = lambda: M.spmv_complex_dev(dA, dxr.data_ptr(), dxi.data_ptr(), dyr.data_ptr(), dyi.data_ptr(),  # noqa
                                          order, stream.cuda_stream)
    else:
        dx = torch.from_numpy(x).to(dev)
        dy = torch.empty((n, K), dtype=torch.float64, device=dev)
        step = lambda: M.spmv_dev(dA, dx.data_ptr(), dy.data_ptr(), order, stream.cuda_stream)  # noqa: E731
    # L2 flush between timed steps: write a 256 MB buffer (> 126 MB L2), then
    # read a second 256 MB buffer so the dirty lines of the write are evicted
    # before the timed launch (the kernel starts with a cold, clean L2 instead
    # of paying for the flush's write-backs)
    flush_w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    flush_r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    flush_acc = torch.zeros(1, dtype=torch.int64, device=dev)

    class _Flush:
        @staticmethod
        def zero_():
            flush_w.zero_()
            flush_acc.add_(flush_r.sum())

    flush = _Flush()
    for _ in range(args.warmup):
        flush.zero_()
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
        flush.zero_()
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = clk.stop()
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_total = sum(ms) / 1e3
    if dist:
        t = torch.tensor([t_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_total = float(t.item())
    per_launch = t_total / args.steps

    # e2e through the host-pointer C-ABI call (pinned host buffers, H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        if cplx:
            hx = [torch.from_numpy(v).pin_memory() for v in x]
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
            flush.zero_()
            ctx.check(call())
        ets = []
        if dist:
            dist.barrier()
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.check(call())
            e1.record(stream)
            torch.cuda.synchronize()
            ets.append(e0.elapsed_time(e1) / 1e3)
        te = sum(ets)
        if dist:
            t = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": world * nnz * args.steps / te / 1e9, "unit": "Gnnz/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}
    launches = args.steps * ((1 if st.nslices > 0 else 0) + (1 if st.nlong > 0 else 0))
    res = dict(n=n, nnz=nnz, t_total=t_total, per_launch=per_launch, clocks=clocks, e2e=e2e, launches=launches,
               stats=st, ctx=ctx, cplx=cplx)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--K", type=int, default=4)
    ap.add_argument("--order", default="fast", choices=["fast", "lane4", "scalar"])
    ap.add_argument("--all", action="store_true", help="one line per config/precision (not the driver line)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--secondary", default="", help="extra K to report beside the headline (default: TD for cfg2)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    order = {"fast": 2, "lane4": 1, "scalar": 0}[args.order]

    if args.impl == "reference":
        if rank != 0:
            return 0
        r = run_reference(args, args.config, args.K)
        line = {"metric": METRIC, "value": r["value"], "unit": "Gnnz/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["median_s"] * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference",
                "config": {"workload": f"{args.config} {K_NAME[args.K]}: {CONFIG_DESC[args.config]}",
                           "precision": K_NAME[args.K], "order": "lane4 (reference default)"},
                "cpu_baseline": {"value": r["value"], "unit": "Gnnz/s", "cores": r["cores"], "kind": r["kind"],
                                 "sample": r["sample"]},
                "e2e": {"value": r["value"], "unit": "Gnnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch

    dist = None
    if world > 1:
        import torch.distributed as tdist

        torch.cuda.set_device(local)
        tdist.init_process_group("nccl")
        dist = tdist
    else:
        torch.cuda.set_device(0)

    import paper_2412_17510_b200 as M

    hbm_peak, hbm_src = measured_peaks()
    probe = M.Context(torch.cuda.current_device())
    fp64_peak = M.measure_fp64_peak(probe)
    probe.close()

    jobs = [(args.config, args.K)]
    if args.all:
        jobs = [("cfg1", 2), ("cfg2", 3), ("cfg2", 4), ("cfg3", 2), ("cfg3", 4), ("cfg4", 2), ("cfg5", 2), ("cfg5", 4)]
    secondary = None
    if not args.all and args.config == "cfg2" and args.K == 4 and args.secondary != "none":
        secondary = ("cfg2", 3)

    def describe(cfg, K, r):
        cplx = r["cplx"]
        nnz, n = r["nnz"], r["n"]
        byts = algorithmic_bytes(nnz, n, K, cplx)
        ops = algorithmic_ops(nnz, K, cplx)
        t_hbm, t_fp = byts / (hbm_peak * 1e9), ops / fp64_peak
        bound = "hbm" if t_hbm >= t_fp else "fp64"
        if bound == "hbm":
            ach = byts / r["per_launch"] / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                    "peak_source": hbm_src}
        else:
            ach = ops / r["per_launch"] / 1e12
            pk = fp64_peak / 1e12
            roof = {"bound": "fp64", "achieved": ach, "peak": pk, "unit": "Tops/s (fp64 instr)", "frac": ach / pk,
                    "peak_source": "measured on this GPU by mpsg_measure_fp64_peak (DFMA throughput)"}
        roof["t_roofline_us"] = max(t_hbm, t_fp) * 1e6
        roof["algorithmic_bytes"] = byts
        roof["algorithmic_fp64_ops"] = ops
        roof["traffic"] = traffic_for(cfg, K)
        return roof

    results = []
    for cfg, K in jobs + ([secondary] if secondary else []):
        r = run_gpu(args, cfg, K, order, rank, world, dist)
        r["roof"] = describe(cfg, K, r)
        results.append((cfg, K, r))
        r["ctx"].close()

    if rank == 0:
        for idx, (cfg, K, r) in enumerate(results[: len(jobs)]):
            value = world * r["nnz"] * args.steps / r["t_total"] / 1e9
            line = {"metric": METRIC, "value": value, "unit": "Gnnz/s", "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": r["t_total"] / args.steps * 1e3,
                    "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic (seeded generators, synth/mpsgen.c)",
                    "config": {"workload": f"{cfg} {K_NAME[K]}: {CONFIG_DESC[cfg]}", "precision": K_NAME[K],
                               "order": args.order, "nnz": r["nnz"], "n": r["n"],
                               "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                               "l2": "flushed before every timed step: 256 MB write, then 256 MB read of a second buffer"},
                    "roofline": r["roof"], "clocks": r["clocks"], "e2e": r["e2e"], "gpu_launches": r["launches"]}
            if secondary and idx == 0:
                c2, k2, r2 = results[-1]
                line["secondary"] = {"workload": f"{c2} {K_NAME[k2]}",
                                     "value": world * r2["nnz"] * args.steps / r2["t_total"] / 1e9,
                                     "unit": "Gnnz/s", "roofline": r2["roof"],
                                     "e2e": r2["e2e"]}
            if world == 1 and not args.no_cpu and not args.all:
                cb = run_reference(argparse.Namespace(steps=5, warmup=1), cfg, K)
                line["cpu_baseline"] = {"value": cb["value"], "unit": "Gnnz/s", "cores": cb["cores"],
                                        "kind": cb["kind"], "sample": cb["sample"]}
            print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def traffic_for(cfg, K):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{cfg}_K{K}")
    return None


if __name__ == "__main__":
    sys.exit(main())
