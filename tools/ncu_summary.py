#!/usr/bin/env python
"""Summarise ncu artefacts from gpurun_out/ into profiles/ (run here, no GPU).

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/<name>_launches.txt
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep      > profiles/<name>_ncu.txt
"""
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "smsp__warps_eligible.avg.per_cycle_active", "sm__cycles_active.avg"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = {}
    print(f"# per-launch device time (ncu --metrics gpu__time_duration.sum --clock-control none) from {path}")
    print("# cold-cache, serialised: compare shares, not absolutes")
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"]
            val = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            ns = val * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
            print(f"{d['ID']:>4}  {ns / 1e3:10.2f} us  {name[:110]}")
            key = name.split("(")[0]
            tot[key] = tot.get(key, 0.0) + ns
    s = sum(tot.values())
    print("\n# share of total device time by kernel")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{100 * v / s:6.1f}%  {v / 1e3:10.1f} us  {k[:100]}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"\n## kernel: {d.get('Kernel Name', '?')[:140]}")
        for k in RAW:
            if k in hdr:
                print(f"  {k:70s} {d[k]} {units[hdr.index(k)]}")
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    print("\n# details page (section | metric | unit | value)")
    for r in csv.reader(io.StringIO(det)):
        if len(r) >= 4 and r[-4] not in ("Section Name",) and not r[-4].startswith(("OPT", "INF", "WRN")):
            if r[-4] in ("PM Sampling",):
                continue
            print(f"  {r[-4]} | {r[-3]} | {r[-2]} | {r[-1]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
