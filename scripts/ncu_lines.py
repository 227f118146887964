#!/usr/bin/env python
"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump (gzip) by CUDA source
line: executed warp instructions, thread instructions (divergence = avg active threads) and
warp-stall samples per unit of work.

usage: python scripts/ncu_lines.py gpurun_out/src_TAG.csv.gz UNITS [TOP]"""
import csv
import gzip
import io
import sys

path, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(io.TextIOWrapper(gzip.open(path), encoding="utf-8")))
file_, hdr, stats = None, None, {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        file_ = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or not r[0]:
        continue  # sass rows (no line number) are included in their cuda line's totals
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ex = int(d.get("Instructions Executed") or 0)
        th = int(d.get("Thread Instructions Executed") or 0)
        st = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    key = (file_, int(r[0]))
    a = stats.setdefault(key, [0, 0, 0, r[1][:70]])
    a[0] += ex
    a[1] += th
    a[2] += st
tot = sum(v[0] for v in stats.values()) or 1
tst = sum(v[2] for v in stats.values()) or 1
print(f"total warp instructions per unit {tot / units:.2f}")
print(f"{'file:line':28s} {'inst/unit':>9s} {'share':>6s} {'thr/inst':>8s} {'stall%':>6s}  source")
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0] + ':' + str(k[1]):28s} {v[0] / units:9.3f} {100 * v[0] / tot:5.1f}% "
          f"{v[1] / max(1, v[0]):8.1f} {100 * v[2] / tst:5.1f}%  {v[3]}")
