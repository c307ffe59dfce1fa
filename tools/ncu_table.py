#!/usr/bin/env python
"""One line per kernel of an ncu --set full report (run here, no GPU):
    python tools/ncu_table.py gpurun_out/prof_all.ncu-rep [labels...]"""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB", None),
        ("dram__bytes_write.sum", "MB", None), ("launch__registers_per_thread", "regs", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%", 1),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%", 1),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1)]


def mb(v, unit):
    f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(unit, 1)
    return v * f


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        vals = []
        for k, lab, scale in COLS:
            v = float(d[k].replace(",", "")) if k in d and d[k] else float("nan")
            u = units[hdr.index(k)] if k in hdr else ""
            if lab == "MB":
                v = mb(v, u)
            elif lab == "us":
                v = v * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(u, 1)
            vals.append(v)
        yield d.get("Kernel Name", "?"), vals


if __name__ == "__main__":
    labels = sys.argv[2:]
    print(f"# {sys.argv[1]}: one row per profiled launch (ncu --set full, cold caches, clocks not locked)")
    print("# " + " | ".join(["label", "kernel"] + [c[1] for c in COLS]) + " | traffic MB = read + write")
    i = 0
    for name, v in rows(sys.argv[1]):
        short = name.split("(")[0].replace("void ", "").replace("mpsg::", "")
        if short.startswith("<unnamed>"):
            continue
        lab = labels[i] if i < len(labels) else ""
        i += 1
        print(f"{lab:10s} | {short:40s} | {v[0]:9.1f} | {v[1]:9.1f} | {v[2]:7.1f} | {int(v[3]):3d} | "
              f"{v[4]:5.1f} | {v[5]:5.1f} | {v[6]:5.1f} | {v[7]:5.1f} | {v[1] + v[2]:9.1f}")
