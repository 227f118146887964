"""The command line against the reference CLI's own outputs (tests/golden/cli.json, made by
tests/golden/make_golden_cli.py running cipherclimb/cli.py).  Reports must be identical
except the `timing` block / elapsed line / wall_ms column (reference tests/test_cli.py
:119-143, :219-238)."""
import contextlib
import io
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2103_13937_b200 as cc
from paper_2103_13937_b200 import cli

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "cli.json").read_text())


def _inputs(d: Path, golden):
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    from make_golden_cli import write_inputs

    write_inputs(d, cc.format_bigram_file, cc.BigramTable(golden.english_scores()),
                 golden.plain_mas(637), golden.plain_sct(596), cc.mas_encrypt, cc.sct_encrypt,
                 cc.demap)


def _run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            code = cli.main(argv)
        except SystemExit as e:
            code = e.code
    return code, out.getvalue(), err.getvalue()


def _case(i, tmp_path, golden):
    _inputs(tmp_path, golden)
    c = GOLDEN[i]
    code, out, err = _run([a.replace("{dir}", str(tmp_path)) for a in c["argv"]])
    return c, code, out.replace(str(tmp_path), "{dir}"), err.replace(str(tmp_path), "{dir}")


def _gpu_case(c):
    return c["argv"][0] in ("solve", "benchmark") and c["code"] == 0 or "--random-key" in c["argv"]


CPU_CASES = [i for i, c in enumerate(GOLDEN) if not _gpu_case(c)]
GPU_CASES = [i for i, c in enumerate(GOLDEN) if _gpu_case(c)]


def test_bigram_file_format_matches_reference_sha(tmp_path, golden):
    _inputs(tmp_path, golden)
    rep = json.loads(GOLDEN[0]["stdout"])
    import hashlib

    assert hashlib.sha256((tmp_path / "bigrams.txt").read_bytes()).hexdigest() == \
        rep["inputs"]["bigrams_sha256"]


@pytest.mark.parametrize("i", CPU_CASES)
def test_cli_host_commands(i, tmp_path, golden):
    c, code, out, err = _case(i, tmp_path, golden)
    assert code == c["code"]
    if c["argv"][0] == "solve" and "bogus" in c["argv"]:
        assert err.startswith("usage: cipherclimb solve") and "invalid choice" in err
        return
    assert out == c["stdout"] and err == c["stderr"]
    if "file" in c:
        assert (tmp_path / "out_bigrams.txt").read_text() == c["file"]


@pytest.mark.gpu
@pytest.mark.parametrize("i", GPU_CASES)
def test_cli_gpu_commands(i, tmp_path, golden):
    c, code, out, err = _case(i, tmp_path, golden)
    assert code == c["code"]
    argv = c["argv"]
    if argv[0] == "solve" and "json" in argv:
        got, want = json.loads(out), json.loads(c["stdout"])
        assert set(got["timing"]) == set(want["timing"])
        got.pop("timing"), want.pop("timing")
        assert got == want
    elif argv[0] == "solve":
        strip = lambda s: [ln for ln in s.splitlines() if not ln.startswith("elapsed:")]
        assert strip(out) == strip(c["stdout"])
    elif argv[0] == "benchmark":
        cols = lambda s: [ln.split(",")[:5] + ln.split(",")[6:] for ln in s.splitlines()]
        assert cols(out) == cols(c["stdout"])
    else:
        assert out == c["stdout"] and err == c["stderr"]
