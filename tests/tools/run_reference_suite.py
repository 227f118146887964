#!/usr/bin/env python
"""Run the reference's OWN test-suite (pkg/tests of /root/reference, 127 tests) against this
repo's GPU engine with `cipherclimb` aliased to paper_2103_13937_b200 (tests/tools/
ref_alias_plugin.py) -- the drop-in claim of INTEGRATION.md section 1, exercised.

The reference tree exists only in the build container and the engine needs a GPU, so the
run has two steps:
  1. here:        python tests/tools/run_reference_suite.py --stage
     copies the reference's tests/ and data/ into oracle/_ref/pkg/ (git-ignored, never
     committed -- the same scratch area as other reference artefacts; it travels to the GPU
     box with the gpurun snapshot);
  2. on the box:  python tests/tools/run_reference_suite.py --run [pytest args]
     runs them (subprocess CLI tests get the alias through PYTHONPATH's sitecustomize).
The pytest summary is written to gpurun_out/reference_suite.txt.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
STAGE = ROOT / "oracle" / "_ref" / "pkg"
REF = Path("/root/reference/pkg")


def stage():
    if STAGE.exists():
        shutil.rmtree(STAGE)
    STAGE.mkdir(parents=True)
    shutil.copytree(REF / "tests", STAGE / "tests")
    shutil.copytree(REF / "data", STAGE / "data")
    print("staged", sorted(p.name for p in (STAGE / "tests").glob("*.py")))


def run(extra):
    tools = ROOT / "tests" / "tools"
    shim = STAGE / "_alias"  # sitecustomize for the subprocess CLI test (python -m cipherclimb.cli)
    shim.mkdir(exist_ok=True)
    (shim / "sitecustomize.py").write_text("import ref_alias_plugin  # noqa: F401\n")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(tools), str(shim)])
    cmd = [sys.executable, "-m", "pytest", str(STAGE / "tests"), "-p", "ref_alias_plugin",
           "-p", "no:cacheprovider", "-q", "-rfE", "--rootdir", str(STAGE), *extra]
    r = subprocess.run(cmd, cwd=str(STAGE), env=env, capture_output=True, text=True)
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / "reference_suite.txt").write_text(
        "$ " + " ".join(cmd) + "\n\n" + r.stdout[-60000:] + "\n" + r.stderr[-5000:])
    print(r.stdout[-3000:])
    return r.returncode


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--stage":
        stage()
    elif len(sys.argv) > 1 and sys.argv[1] == "--run":
        sys.exit(run(sys.argv[2:]))
    else:
        print(__doc__)
