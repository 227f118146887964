"""pytest plugin: make `import cipherclimb` (and every cipherclimb.<module>) resolve to this
repo's GPU engine, so the reference's own test-suite runs against the drop-in unchanged
(INTEGRATION.md section 1).  Loaded with `-p ref_alias_plugin` by run_reference_suite.py."""
import importlib
import sys

MODULES = ("codec", "ngrams", "rng", "ciphers", "pairs", "search", "mas", "sct", "cli")


def install():
    pkg = importlib.import_module("paper_2103_13937_b200")
    sys.modules["cipherclimb"] = pkg
    for m in MODULES:
        sys.modules[f"cipherclimb.{m}"] = importlib.import_module(f"paper_2103_13937_b200.{m}")


install()
