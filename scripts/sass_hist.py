#!/usr/bin/env python
"""Histogram of a kernel's executed SASS by execution count (ncu source page):
usage: sass_hist.py REPORT.ncu-rep UNITS [top]   (UNITS = tries in the capture)"""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows, h = [], None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        h = None
        continue
    if r and r[0] == "Address":
        h = r
        continue
    if h:
        rows.append(dict(zip(h, r)))
b = collections.defaultdict(lambda: [0.0, 0, 0, collections.Counter()])
tot_s = 0
tot = 0.0
for r in rows:
    v = int(r.get("Instructions Executed") or 0)
    if not v:
        continue
    s = int(r.get("Warp Stall Sampling (All Samples)") or 0)
    tot_s += s
    tot += v / units
    k = round(v / units, 3)
    op = r["Source"].split()
    op = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "")
    b[k][0] += v / units
    b[k][1] += 1
    b[k][2] += s
    b[k][3][op] += 1
print(f"total executed warp instructions per unit: {tot:.2f}")
print(f"{'execs/unit':>10} {'#inst':>6} {'inst/unit':>9} {'stall%':>6}  opcodes")
for k, (v, c, s, ops) in sorted(b.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{k:10.3f} {c:6d} {v:9.2f} {100 * s / max(1, tot_s):6.1f}  {dict(ops.most_common(7))}")
