"""Loaders for tests/golden/*.npz (reference outputs frozen by tests/golden/make_golden.py)
plus the input recipes those outputs were produced from, so tests can rebuild the
inputs on a box without /root/reference."""
from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
KEYGEN_STREAM = 2**32 - 2


@lru_cache(maxsize=None)
def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def data():
    return load("data")


def english_scores() -> np.ndarray:
    return data()["english_scores"].astype(np.int64)


def english_logs() -> np.ndarray:
    return data()["english_logs"].astype(np.float64)


def plain_mas(n=471) -> np.ndarray:
    return data()["plain_mas"][:n].astype(np.int64)


def plain_sct(n=596) -> np.ndarray:
    return data()["plain_sct"][:n].astype(np.int64)


def corpus() -> np.ndarray:
    return data()["corpus"].astype(np.int64)


def scoring_texts():
    g = load("scoring")
    return [np.random.default_rng(900 + i).integers(0, 26, int(L)) for i, L in enumerate(g["lengths"])]


def delta_cases():
    """Acceptance #05 recipe (reference tests/test_acceptance.py:113-124)."""
    rng = np.random.default_rng(501)
    table = rng.integers(0, 900, 676)
    cases = []
    for _ in range(10_000):
        text = rng.integers(0, 26, int(rng.integers(2, 220)))
        a, b = (int(v) for v in rng.choice(26, size=2, replace=False))
        cases.append((text, a, b))
    return table, cases, load("mas_delta")["deltas"]


def _mas_table(tid):
    g = load("mas_workers")
    return {0: english_scores(), 1: g["table1"], 2: g["table2"]}[int(tid)]


def mas_worker_cases(permutation):
    """[(cipher, table, climbings, seed, stream, want_text, want_score)].

    `permutation(seed, stream, n)` must be the reference-exact Philox permutation
    (oracle or engine) -- the ciphertext keys were drawn with it on KEYGEN_STREAM."""
    g = load("mas_workers")
    out = []
    pos = 0
    pm, cp = data()["plain_mas"].astype(np.int64), corpus()
    for i in range(g["score"].size):
        L = int(g["lengths"][i])
        src = cp if g["src_corpus"][i] else pm
        off = int(g["offsets_src"][i])
        plain = src[off:off + L]
        key = permutation(int(g["key_seed"][i]), KEYGEN_STREAM, 26)
        cipher = key[plain]
        want = g["text"][pos:pos + L].astype(np.int64)
        pos += L
        out.append((cipher, _mas_table(g["table_id"][i]), int(g["climbings"][i]), int(g["seed"][i]),
                    int(g["stream"][i]), want, int(g["score"][i])))
    return out


def sct_worker_cases():
    """[(cipher, logs, k, climbings, seed, stream, want_key, want_score)]."""
    g = load("sct_workers")
    out = []
    pk = pc = 0
    for i in range(g["score"].size):
        k, n = int(g["k"][i]), int(g["n"][i])
        logs = english_logs() if int(g["table_id"][i]) == 0 else g["tiny_logs"]
        cipher = g["cipher"][pc:pc + n].astype(np.int64)
        key = g["key"][pk:pk + k].astype(np.int64)
        pc += n
        pk += k
        out.append((cipher, logs, k, int(g["climbings"][i]), int(g["seed"][i]), int(g["stream"][i]),
                    key, float(g["score"][i])))
    return out


def gather_cases(permutation):
    g = load("sct_gather")
    out = []
    pos = 0
    for k, n in g["cases"]:
        key = permutation(int(k) * 1000 + int(n), 0, int(k))
        out.append((key, int(n), g["maps"][pos:pos + n]))
        pos += n
    return out


def det_step_cases():
    """[(text, (pl, pr), table, want_score, want_index, want_candidate)] from
    tests/golden/mas_det.npz (reference deterministic_step, mas.py:84-120)."""
    g = load("mas_det")
    out, pos = [], 0
    for i, L in enumerate(g["step_len"]):
        L = int(L)
        text = g["step_text"][pos:pos + L].astype(np.int64)
        cand = g["step_cand"][pos:pos + L].astype(np.int64)
        pos += L
        pl, pr = (int(v) for v in g["step_pivot"][i])
        out.append((text, (pl, pr), g["tables"][int(g["step_table"][i])], int(g["step_score"][i]),
                    int(g["step_index"][i]), cand))
    return out


def det_run_cases():
    """[(cipher, table, seed, restart, iterations, want_text, want_score, want_history)] from
    reference solve_deterministic runs (mas.py:140-169)."""
    g = load("mas_det")
    out, pos, hpos = [], 0, 0
    for i, L in enumerate(g["run_len"]):
        L = int(L)
        nh = int(g["run_nhist"][i])
        hist = [(int(a), int(b)) for a, b in g["run_hist"][hpos:hpos + nh]]
        hpos += nh
        out.append((g["run_cipher"][pos:pos + L].astype(np.int64), g["tables"][int(g["run_table"][i])],
                    int(g["run_seed"][i]), int(g["run_restart"][i]), int(g["run_iters"][i]),
                    g["run_text"][pos:pos + L].astype(np.int64), int(g["run_score"][i]), hist))
        pos += L
    return out
