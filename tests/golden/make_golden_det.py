"""Golden fixtures for the deterministic best-neighbour MAS solver (reference mas.py:84-169),
produced by running the REFERENCE itself.  Run in the dev container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_det.py

Writes tests/golden/mas_det.npz:
  step_*   acceptance #04's recipe (tests/test_acceptance.py:73-110: default_rng(401), table
           integers(0, 600), 100 texts of 200 letters, pivots drawn with rng.choice) plus
           test_mas.py:85-95's recipe (default_rng(9), table default_rng(10) integers(0,500));
           outputs of cipherclimb.deterministic_step: best score, best index, candidate text.
  run_*    cipherclimb.solve_deterministic runs: acceptance #06's input (plain_mas[:471],
           key WorkerRng(600, KEYGEN).permutation(26), seed 606, 500 iterations) for
           restarts 0..3, and random ciphertexts/tables of other lengths and budgets;
           outputs: best_text, best_score, history (iteration, score).
"""
from __future__ import annotations

import time
from pathlib import Path

import numpy as np

import cipherclimb as cc
from cipherclimb.rng import KEYGEN_STREAM

OUT = Path(__file__).resolve().parent
DATA = Path("/root/reference/pkg/data")
t0 = time.time()

# ----------------------------------------------------------------- deterministic_step
step_text, step_pl, step_pr, step_table, step_score, step_index, step_cand = [], [], [], [], [], [], []
tables = []
rng = np.random.default_rng(401)
tables.append(rng.integers(0, 600, 676))
for _ in range(100):
    text = rng.integers(0, 26, 200)
    present = np.unique(text)
    pl, pr = (int(v) for v in rng.choice(present, size=2, replace=False))
    cand, score, index = cc.deterministic_step(text, (pl, pr), cc.BigramTable(tables[0]))
    step_text.append(text); step_pl.append(pl); step_pr.append(pr); step_table.append(0)
    step_score.append(score); step_index.append(index); step_cand.append(cand)
tables.append(np.random.default_rng(10).integers(0, 500, 676))
rng = np.random.default_rng(9)
for _ in range(20):
    text = rng.integers(0, 26, 200)
    present = np.unique(text)
    pl, pr = (int(v) for v in rng.choice(present, size=2, replace=False))
    cand, score, index = cc.deterministic_step(text, (pl, pr), cc.BigramTable(tables[1]))
    step_text.append(text); step_pl.append(pl); step_pr.append(pr); step_table.append(1)
    step_score.append(score); step_index.append(index); step_cand.append(cand)
# short texts, few present letters, pivots at the alphabet ends (exclusion edge cases)
rng = np.random.default_rng(4242)
tables.append(rng.integers(0, 60_000, 676))
for i in range(40):
    L = int(rng.integers(2, 40))
    alpha = rng.choice(26, size=int(rng.integers(2, 6)), replace=False)
    text = alpha[rng.integers(0, alpha.size, L)]
    present = np.unique(text)
    if present.size < 2:
        text[0], text[-1] = alpha[0], alpha[1]
        present = np.unique(text)
    pl, pr = (int(v) for v in rng.choice(present, size=2, replace=False))
    cand, score, index = cc.deterministic_step(text, (pl, pr), cc.BigramTable(tables[2]))
    step_text.append(text); step_pl.append(pl); step_pr.append(pr); step_table.append(2)
    step_score.append(score); step_index.append(index); step_cand.append(cand)
print(f"[{time.time() - t0:6.1f}s] {len(step_score)} deterministic_step cases", flush=True)

# ----------------------------------------------------------------- solve_deterministic
english = cc.parse_bigram_file((DATA / "english_bigrams.txt").read_text())
plain_mas = cc.map_text(cc.normalize((DATA / "sample_plain_mas.txt").read_text()))[:471]
runs = []  # (cipher, table_id, seed, restart, iterations)
key = cc.WorkerRng(600, KEYGEN_STREAM).permutation(26)
c06 = cc.mas_encrypt(plain_mas, key)
tables.append(english.scores)  # id 3
for r in range(4):
    runs.append((c06, 3, 606, r, 500))
rng = np.random.default_rng(77)
for i, (L, iters) in enumerate([(2, 300), (3, 300), (17, 300), (60, 300), (150, 1), (150, 300),
                                (300, 500), (800, 100), (1500, 40), (40, 7)]):
    cipher = rng.integers(0, 26, L)
    if np.unique(cipher).size < 2:
        cipher[0], cipher[-1] = 1, 2
    tid = int(rng.integers(0, 3)) if i % 2 else 3
    runs.append((cipher, tid, int(rng.integers(0, 2**63)), int(rng.integers(0, 5)), iters))

run_cipher, run_text, run_hist = [], [], []
run_len, run_table, run_seed, run_restart, run_iters, run_score, run_nhist = ([] for _ in range(7))
for cipher, tid, seed, r, iters in runs:
    cfg = cc.MasSolverConfig(mode="deterministic", workers=325, iterations=iters, global_seed=seed)
    res = cc.solve_deterministic(cipher, cc.BigramTable(tables[tid]), cfg, restart=r)
    run_cipher.append(np.asarray(cipher)); run_text.append(res.best_text)
    run_hist.extend(res.history); run_nhist.append(len(res.history))
    run_len.append(len(cipher)); run_table.append(tid); run_seed.append(seed)
    run_restart.append(r); run_iters.append(iters); run_score.append(res.best_score)
    print(f"[{time.time() - t0:6.1f}s] run L={len(cipher)} iters={iters} r={r} "
          f"score={res.best_score} accepts={len(res.history)}", flush=True)

np.savez_compressed(
    OUT / "mas_det.npz",
    tables=np.array(tables, dtype=np.int64),
    step_len=np.array([t.size for t in step_text]),
    step_text=np.concatenate(step_text).astype(np.uint8),
    step_pivot=np.array([step_pl, step_pr]).T,
    step_table=np.array(step_table),
    step_score=np.array(step_score, dtype=np.int64),
    step_index=np.array(step_index),
    step_cand=np.concatenate(step_cand).astype(np.uint8),
    run_len=np.array(run_len), run_cipher=np.concatenate(run_cipher).astype(np.uint8),
    run_table=np.array(run_table), run_seed=np.array(run_seed, dtype=np.uint64),
    run_restart=np.array(run_restart), run_iters=np.array(run_iters),
    run_score=np.array(run_score, dtype=np.int64), run_text=np.concatenate(run_text).astype(np.uint8),
    run_nhist=np.array(run_nhist), run_hist=np.array(run_hist, dtype=np.int64).reshape(-1, 2),
)
print(f"[{time.time() - t0:6.1f}s] wrote {OUT / 'mas_det.npz'}")
