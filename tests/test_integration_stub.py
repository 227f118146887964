"""INTEGRATION.md section 2, executed: the reference-side ctypes stub
(integration/cipherclimb_b200_stub.py, dropped into the reference as cipherclimb/_b200.py)
run on task tuples built exactly as the reference builds them (mas.py:266-270,
sct.py:194-198) reproduces the reference's own solve outputs frozen in tests/golden/."""
import importlib.util
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _stub():
    spec = importlib.util.spec_from_file_location(
        "cipherclimb_b200_stub", ROOT / "integration" / "cipherclimb_b200_stub.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@dataclass
class _SctCfg:  # the fields of the reference's SctSolverConfig the stub reads (sct.py:43-55)
    key_length: int
    climbings: int = 15_000
    p1: int = 33
    p2: int = 66
    op1_hop: int = 3
    op2_hop: int = 3


def test_stub_imports_without_the_engine_package():
    """The stub binds the C ABI with ctypes + numpy only (a reference maintainer has no
    paper_2103_13937_b200 package); loading it must not touch the GPU."""
    src = (ROOT / "integration" / "cipherclimb_b200_stub.py").read_text()
    assert "paper_2103_13937_b200" not in src.split('"""', 2)[2]
    m = _stub()
    assert m._lib is None and {"run_stochastic_pool", "run_sct_pool"} <= set(dir(m))


@pytest.mark.gpu
def test_stub_reproduces_reference_mas_solve(golden):
    m = _stub()
    m.load(str(ROOT / "paper_2103_13937_b200" / "libcipherclimb_b200.so"))
    g = golden.load("mas_solve")
    cipher = g["cipher"].astype(np.int64)
    scores = golden.english_scores()
    for r in range(2):
        tasks = [(cipher, scores, 10_000, 7000, (r << 32) | w) for w in range(64)]  # mas.py:266-270
        outcomes = m.run_stochastic_pool(tasks)
        per_worker = [s for _, s in outcomes]
        assert per_worker == g["per_worker"][r].tolist()
        best = int(np.argmax(per_worker))  # search.py:19-25 max_element
        assert np.array_equal(outcomes[best][0], g["best_text"][r])


@pytest.mark.gpu
def test_stub_reproduces_reference_sct_solve(golden):
    m = _stub()
    m.load(str(ROOT / "paper_2103_13937_b200" / "libcipherclimb_b200.so"))
    g = golden.load("sct_solve")
    cipher = g["cipher"].astype(np.int64)
    logs = golden.english_logs()
    cfg = _SctCfg(key_length=10)
    tasks = [(cipher, logs, -24.0, cfg, 8000, w) for w in range(64)]  # sct.py:194-198, r = 0
    outcomes = m.run_sct_pool(tasks)
    per_worker = [s for _, s in outcomes]
    assert per_worker == g["per_worker"].tolist()
    best = int(np.argmax(per_worker))
    assert np.array_equal(outcomes[best][0], g["best_key"])
