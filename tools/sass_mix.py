#!/usr/bin/env python
"""Dynamic SASS mix + stall samples per opcode from an ncu source-page export:
    ncu -i rep --page source --csv --print-source sass > src.csv
    python tools/sass_mix.py src.csv "sell_real_kernel<4, 0>" [nth]"""
import csv
import sys
from collections import defaultdict

path, pat = sys.argv[1], sys.argv[2]
nth = int(sys.argv[3]) if len(sys.argv) > 3 else 0
sections, cur = [], None
hdr = None
for row in csv.reader(open(path)):
    if row and row[0] == "Kernel Name":
        cur = [row[1], []]
        sections.append(cur)
        hdr = None
        continue
    if row and row[0] == "Address":
        hdr = row
        continue
    if cur is not None and hdr and len(row) == len(hdr):
        cur[1].append(dict(zip(hdr, row)))
match = [s for s in sections if pat in s[0]]
name, rows = match[nth]
ex, st, tot = defaultdict(float), defaultdict(float), 0.0
stall_cols = [h for h in hdr if h.startswith("stall_")]
reasons = defaultdict(float)
for r in rows:
    op = r["Source"].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.rstrip(";").split(".")[0]
    n = float(r["Instructions Executed"] or 0)
    ex[o] += n
    tot += n
    st[o] += float(r["Warp Stall Sampling (All Samples)"] or 0)
    for c in stall_cols:
        try:
            reasons[c] += float(r[c] or 0)
        except ValueError:
            pass
print(f"# {name[:100]}  total warp-instructions {tot:.0f}")
fp = sum(v for k, v in ex.items() if k in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"))
print(f"# fp64-pipe ops {fp:.0f} ({100 * fp / tot:.1f}%)")
ss = sum(st.values())
for o, v in sorted(ex.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{o:12s} {v:14.0f} {100 * v / tot:6.2f}%   stall samples {100 * st[o] / max(ss, 1):5.1f}%")
rs = sum(reasons.values())
print("# stall reasons:", ", ".join(f"{k[6:]} {100 * v / rs:.1f}%" for k, v in sorted(reasons.items(), key=lambda kv: -kv[1])[:8]))
