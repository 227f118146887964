"""Golden outputs of the reference command line (cipherclimb/cli.py), produced by running
the REFERENCE itself.  Run in the dev container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cli.py

Writes tests/golden/cli.json: for each case the argv (with {dir} standing for the scratch
directory holding the inputs), the exit code, stdout and stderr.  The inputs are rebuilt
by tests/test_cli.py from tests/golden/data.npz with the same recipe (CASES_INPUTS below):
the bigram file is the english table in the reference's own file format, the ciphertexts
are encryptions of the held-out sample plaintext.
"""
from __future__ import annotations

import contextlib
import io
import json
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
DATA = Path("/root/reference/pkg/data")


def write_inputs(d: Path, fmt, table, plain_mas, plain_sct, mas_encrypt, sct_encrypt, demap):
    """The recipe shared with tests/test_cli.py."""
    (d / "bigrams.txt").write_text(fmt(table))
    key = np.array([(7 * i + 3) % 26 for i in range(26)])
    (d / "mas.txt").write_text(demap(mas_encrypt(plain_mas[:150], key)) + "\n")
    (d / "sct.txt").write_text(demap(sct_encrypt(plain_sct[:240], np.array([3, 0, 5, 1, 4, 2]))) + "\n")
    (d / "plain.txt").write_text(demap(plain_sct[:200]) + "\n")
    (d / "corpus.txt").write_text("The quick brown fox jumps over the lazy dog.\nPack my box!\n")
    (d / "config.json").write_text(json.dumps({"workers": 6, "climbings": 900, "restarts": 2}))


CASES = [
    ["solve", "{dir}/mas.txt", "--mode", "mas", "--bigrams", "{dir}/bigrams.txt", "--workers", "8",
     "--climbings", "2000", "--restarts", "3", "--seed", "5", "--format", "json"],
    ["solve", "{dir}/mas.txt", "--mode", "mas", "--bigrams", "{dir}/bigrams.txt", "--workers", "8",
     "--climbings", "2000", "--restarts", "3", "--seed", "5"],
    ["solve", "{dir}/mas.txt", "--mode", "mas-det", "--bigrams", "{dir}/bigrams.txt",
     "--iterations", "60", "--restarts", "2", "--seed", "6", "--format", "json"],
    ["solve", "{dir}/sct.txt", "--mode", "sct", "--bigrams", "{dir}/bigrams.txt", "--key-length", "6",
     "--workers", "8", "--climbings", "1500", "--restarts", "2", "--seed", "7", "--format", "json"],
    ["solve", "{dir}/sct.txt", "--mode", "sct", "--bigrams", "{dir}/bigrams.txt", "--key-length", "6",
     "--workers", "8", "--climbings", "1500", "--seed", "7"],
    ["solve", "{dir}/mas.txt", "--mode", "mas", "--bigrams", "{dir}/bigrams.txt", "--config",
     "{dir}/config.json", "--workers", "4", "--seed", "9", "--format", "json"],
    ["benchmark", "--plaintext", "{dir}/plain.txt", "--bigrams", "{dir}/bigrams.txt", "--key-sizes",
     "4,5,6", "--workers", "8", "--climbings", "800", "--seed", "11", "--format", "csv"],
    ["benchmark", "--plaintext", "{dir}/plain.txt", "--bigrams", "{dir}/bigrams.txt", "--key-sizes",
     "", "--seed", "1", "--format", "csv"],
    ["encrypt", "mas", "{dir}/plain.txt", "--key", "qwertyuiopasdfghjklzxcvbnm"],
    ["encrypt", "sct", "{dir}/plain.txt", "--random-key", "--key-length", "7", "--seed", "3"],
    ["encrypt", "sct", "{dir}/plain.txt", "--key", "2,0,1"],
    ["corpus-build", "{dir}/corpus.txt", "{dir}/out_bigrams.txt"],
    # error paths (exit codes 1 and 2)
    ["solve", "{dir}/sct.txt", "--mode", "sct", "--bigrams", "{dir}/bigrams.txt", "--seed", "1"],
    ["solve", "{dir}/missing.txt", "--mode", "mas", "--bigrams", "{dir}/bigrams.txt", "--seed", "1"],
    ["encrypt", "mas", "{dir}/plain.txt", "--key", "abc"],
    ["solve", "{dir}/mas.txt", "--mode", "bogus", "--bigrams", "{dir}/bigrams.txt"],
]


def run(argv):
    from cipherclimb import cli

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            code = cli.main(argv)
        except SystemExit as e:
            code = e.code
    return code, out.getvalue(), err.getvalue()


if __name__ == "__main__":
    import cipherclimb as cc

    corpus = (DATA / "corpus.txt").read_text()
    table = cc.build_table_from_corpus(corpus)
    pm = cc.map_text(cc.normalize((DATA / "sample_plain_mas.txt").read_text()))
    ps = cc.map_text(cc.normalize((DATA / "sample_plain_sct.txt").read_text()))
    results = []
    with tempfile.TemporaryDirectory() as tmp:
        d = Path(tmp)
        write_inputs(d, cc.format_bigram_file, table, pm, ps, cc.mas_encrypt, cc.sct_encrypt, cc.demap)
        for argv in CASES:
            code, out, err = run([a.replace("{dir}", tmp) for a in argv])
            extra = {}
            if argv[0] == "corpus-build" and code == 0:
                extra["file"] = (d / "out_bigrams.txt").read_text()
            results.append({"argv": argv, "code": code, "stdout": out.replace(tmp, "{dir}"),
                            "stderr": err.replace(tmp, "{dir}"), **extra})
            print(argv[:3], code)
    (OUT / "cli.json").write_text(json.dumps(results, indent=1))
    print("wrote", OUT / "cli.json")
