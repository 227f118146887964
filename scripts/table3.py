#!/usr/bin/env python
"""Replicate the paper's only published GPU table (Table 3: SCT solve of
the 596-letter sample text, k = 10..35, 1120 threads x 15k / 30k / 100k climbings, GTX 1060)
on B200 with this repo's CLI `benchmark` command (the reference's cli.py:299-349 with the
same flags), and print one JSON line per row beside the paper's CUDA and CrypTool times.
Inputs are the reference's pkg/data files (frozen in tests/golden/data.npz)."""
import json
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import golden_data as G  # noqa: E402
import paper_2103_13937_b200 as cc  # noqa: E402

PAPER = {10: (15_000, 5.5, "27m"), 15: (15_000, 6.5, "27m"), 20: (15_000, 5.5, "28m"),
         25: (15_000, 5.9, "28m"), 30: (30_000, 10.7, "55m"), 35: (100_000, 46.2, "3h 11m")}


def main():
    tmp = Path(tempfile.mkdtemp())
    plain = "".join(chr(97 + int(x)) for x in G.plain_sct(596))
    (tmp / "plain.txt").write_text(plain)
    (tmp / "bigrams.txt").write_text(cc.format_bigram_file(cc.BigramTable(G.english_scores())))
    seeds = [int(s) for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0"])]
    # each CLI call is a fresh process: a leading k=5 row absorbs the CUDA context and module
    # load and is dropped (the row seeds are --seed + row index, as in the reference CLI)
    for climbings, ks in ((15_000, "5,10,15,20,25"), (30_000, "5,30"), (100_000, "5,35")):
        for seed in seeds:
            cmd = [sys.executable, "-m", "paper_2103_13937_b200.cli", "benchmark", "--plaintext",
                   str(tmp / "plain.txt"), "--bigrams", str(tmp / "bigrams.txt"), "--key-sizes", ks,
                   "--workers", "1120", "--climbings", str(climbings), "--seed", str(seed),
                   "--format", "csv"]
            out = subprocess.run(cmd, capture_output=True, text=True, check=True, cwd=ROOT).stdout
            lines = out.strip().splitlines()
            hdr = lines[0].split(",")
            for row in lines[2:]:
                d = dict(zip(hdr, row.split(",")))
                k = int(d["key_size"])
                pc, pt, ct = PAPER[k]
                d = {"key_size": k, "workers": int(d["workers"]), "climbings": int(d["climbings"]),
                     "seed": int(d["seed"]), "b200_wall_s": int(d["wall_ms"]) / 1e3,
                     "recovered": int(d["recovered"]),
                     "b200_evals_per_s": int(d["workers"]) * int(d["climbings"]) / (int(d["wall_ms"]) / 1e3),
                     "paper_gtx1060_s": pt, "paper_cryptool": ct,
                     "speedup_vs_gtx1060": pt / (int(d["wall_ms"]) / 1e3),
                     "cmd": "python -m paper_2103_13937_b200.cli " + " ".join(cmd[3:])}
                print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
