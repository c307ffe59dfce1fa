#!/usr/bin/env python
"""DRAM traffic per SpMV launch for every bench line (GPU box; development tool).

    python tools/traffic.py [out.json]

For each bench.py --all SpMV line, one ncu process runs ONE SpMV of that line
through tools/kbench.py (--steps 1 --warmup 0, L2 flushed before it) and
collects dram__bytes_read.sum + dram__bytes_write.sum of every SpMV kernel of
that launch (the SELL kernel and, where present, the long-row kernel); the sum
is the line's `roofline.traffic` (profiles/traffic.json, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# bench key -> kbench spec
SPECS = {}
for c, k in [(1, 2), (2, 3), (2, 4), (3, 2), (3, 4), (4, 2), (5, 2), (5, 4)]:
    SPECS[f"cfg{c}_K{k}"] = f"cfg{c}:{k}:2"
    SPECS[f"cfg{c}_K{k}_o1"] = f"cfg{c}:{k}:1"
SPECS.update({"cfg2_K4_mixed": "cfg2:4:2:mixed", "cfg4_K2_mixed": "cfg4:2:2:mixed", "cfg3_K4_mixed": "cfg3:4:2:mixed",
              "cfg2_K4_sptmv": "cfg2:4:2:sptmv", "cfg3_K2_sptmv": "cfg3:2:2:sptmv"})


def measure(spec):
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:^(sell|long|pad)_", "--csv",
           sys.executable, os.path.join(ROOT, "tools", "kbench.py"), "--steps", "1", "--warmup", "0", spec]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900).stdout
    rows = [r for r in csv.reader(io.StringIO(out[out.find('"ID"'):])) if r]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    tot, per = 0.0, []
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        name, metric, unit, val = r[ix["Kernel Name"]], r[ix["Metric Name"]], r[ix["Metric Unit"]], r[ix["Metric Value"]]
        v = float(val.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit)
        if metric.startswith("dram__bytes") and scale:
            tot += v * scale
        if metric == "gpu__time_duration.sum":
            per.append((name.split("(")[0], v, unit))
    return tot, per


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "traffic.json")
    res = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per SpMV launch (every SpMV kernel of the "
                    "launch), one cold launch per line through tools/kbench.py under ncu (tools/traffic.py)"}
    kernels = {}
    for key, spec in SPECS.items():
        try:
            t, per = measure(spec)
        except Exception as e:  # noqa: BLE001
            print(key, "failed:", e, flush=True)
            continue
        res[key] = t
        kernels[key] = per
        print(key, spec, f"{t / 1e9:.4f} GB", per, flush=True)
    res["_kernels"] = kernels
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
