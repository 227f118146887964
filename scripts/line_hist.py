#!/usr/bin/env python
"""Per-CUDA-source-line cost of a kernel from an ncu report (cuda,sass source view).

usage: line_hist.py REPORT.ncu-rep UNITS [top]   (UNITS = tries in the capture)
Prints warp instructions per unit and the share of warp-stall samples for each source line
(summed over every inlined copy), hottest first."""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
inst = collections.Counter()
samp = collections.Counter()
text = {}
path = "?"
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 8 or not r[0]:
        continue
    key = (path, int(r[0]))
    text[key] = r[1].strip()[:80]
    try:
        inst[key] += float(r[7])
        samp[key] += float(r[4])
    except ValueError:
        pass
tot_i = sum(inst.values()) / units
tot_s = sum(samp.values()) or 1
print(f"total warp instructions per unit: {tot_i:.2f}")
for key, _ in sorted(samp.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{inst[key] / units:8.2f} {100 * samp[key] / tot_s:5.1f}%  {key[0]}:{key[1]}  {text[key]}")
