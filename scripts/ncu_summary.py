#!/usr/bin/env python
"""Summarise a gpu_cycle.sh run into profiles/ (the committed evidence).

usage: python scripts/ncu_summary.py TAG [TRIES_IN_CAPTURE]

Reads gpurun_out/{bench_TAG.json, launches_TAG.csv, prof_TAG.ncu-rep} and writes
profiles/TAG_bench.json, profiles/TAG_launches.txt, profiles/TAG_ncu.txt.  The ncu capture
of scripts/gpu_cycle.sh is `bench.py --profile --ciphers 2000` (2000 x 64 workers x 10,000
climbings = 1.28e9 tries in one launch) unless TRIES_IN_CAPTURE says otherwise.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]


def ncu_csv(rep: Path, page: str, extra=()):
    r = subprocess.run(["ncu", "-i", str(rep), "--page", page, "--csv", *extra],
                       capture_output=True, text=True, check=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def launches(tag: str) -> str:
    path = OUT / f"launches_{tag}.csv"
    rows = [r for r in csv.reader(path.open()) if len(r) > 10 and r[0] != "ID"]
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        tot[r[4]] += float(r[-1])
        cnt[r[4]] += 1
    all_ns = sum(tot.values())
    lines = ["ncu --metrics gpu__time_duration.sum --clock-control none, "
             "`python bench.py --profile` (1 warm-up + 1 timed step of the bench workload)",
             "per-launch times are cold-cache and serialised; compare shares", "",
             f"{'kernel':90s} {'launches':>8s} {'total_ns':>14s} {'share':>7s}"]
    for k, v in tot.most_common():
        lines.append(f"{k[:90]:90s} {cnt[k]:8d} {v:14.0f} {100 * v / all_ns:6.2f}%")
    return "\n".join(lines) + "\n"


def full(tag: str, tries: float) -> str:
    rep = OUT / f"prof_{tag}.ncu-rep"
    rows = ncu_csv(rep, "raw")
    h, u, v = rows[0], rows[1], rows[2]
    out = [f"ncu --set full --clock-control none --import-source on (gpurun_out/prof_{tag}.ncu-rep)",
           f"kernel: {v[h.index('Kernel Name')]}", f"tries in the captured launch: {tries:.4g}", ""]
    for m in METRICS:
        if m in h:
            i = h.index(m)
            out.append(f"{m:90s} {v[i]:>22s} {u[i]}")
    if "smsp__inst_executed.sum" in h:
        inst = float(v[h.index("smsp__inst_executed.sum")].replace(",", ""))
        out += ["", f"derived: warp instructions per try = {inst / tries:.2f}"]
    # hottest SASS by warp-stall samples (source page; one section per function)
    try:
        src = ncu_csv(rep, "source", ["--print-source", "sass"])
        rows, hh = [], None
        for r in src:
            if r and r[0] == "Kernel Name":
                hh = None
            elif r and r[0] == "Address":
                hh = r
            elif hh:
                rows.append(dict(zip(hh, r)))
        body = [r for r in rows if int(r.get("Instructions Executed") or 0)]
        tot_samples = sum(int(r.get("Warp Stall Sampling (All Samples)") or 0) for r in body) or 1
        body.sort(key=lambda r: -int(r.get("Warp Stall Sampling (All Samples)") or 0))
        out += ["", "top 25 SASS instructions by warp-stall samples "
                "(execs per unit, share of samples, instruction):"]
        for r in body[:25]:
            out.append(f"  {int(r['Instructions Executed']) / tries:8.4f} "
                       f"{100 * int(r.get('Warp Stall Sampling (All Samples)') or 0) / tot_samples:6.2f}%  "
                       f"{r['Source'].strip()[:80]}")
        # where the issued instructions go: opcode histogram weighted by executions, and the
        # most executed SASS lines
        ops = collections.Counter()
        for r in body:
            txt = r["Source"].strip()
            op = txt.split()[0] if not txt.startswith("@") else txt.split()[1]
            ops[op.split(".")[0]] += int(r["Instructions Executed"])
        tot_exec = sum(ops.values()) or 1
        out += ["", "executed warp instructions by opcode (per unit, share):"]
        for op, c in ops.most_common(24):
            out.append(f"  {op:12s} {c / tries:9.3f} {100 * c / tot_exec:6.2f}%")
        body.sort(key=lambda r: -int(r["Instructions Executed"]))
        out += ["", "top 30 SASS instructions by executions (per unit, instruction):"]
        for r in body[:30]:
            out.append(f"  {int(r['Instructions Executed']) / tries:8.4f}  {r['Source'].strip()[:90]}")
    except Exception as e:  # noqa: BLE001
        out.append(f"(source page unavailable: {e})")
    return "\n".join(out) + "\n"


def main():
    tag = sys.argv[1]
    tries = float(sys.argv[2]) if len(sys.argv) > 2 else 2000 * 64 * 10_000
    name = sys.argv[3] if len(sys.argv) > 3 else tag
    PROF.mkdir(exist_ok=True)
    b = OUT / f"bench_{tag}.json"
    if b.exists() and b.stat().st_size:
        line = json.loads(b.read_text().strip().splitlines()[-1])
        (PROF / f"{name}_bench.json").write_text(json.dumps(line, indent=1) + "\n")
    if (OUT / f"launches_{tag}.csv").exists():
        (PROF / f"{name}_launches.txt").write_text(launches(tag))
    if (OUT / f"prof_{tag}.ncu-rep").exists():
        (PROF / f"{name}_ncu.txt").write_text(full(tag, tries))
    print("wrote", sorted(p.name for p in PROF.glob(f"{name}_*")))


if __name__ == "__main__":
    main()
