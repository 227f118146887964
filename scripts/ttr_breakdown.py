#!/usr/bin/env python
"""Where a time-to-recover solve's milliseconds go (acceptance #07 MAS shape: 471 letters,
64 workers x 10,000 climbings; #08 SCT k=10: 596 letters, 64 x 15,000): the public
solve_with_restarts / solve_sct call with stop-on-plaintext vs one engine call for the same
restart, host-timed after warm-up."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import golden_data as G  # noqa: E402
import paper_2103_13937_b200 as cc  # noqa: E402
from paper_2103_13937_b200 import engine  # noqa: E402
from paper_2103_13937_b200.rng import philox_keys  # noqa: E402


def best_of(f, n=20):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), 1e3 * float(np.median(ts))


KEYGEN = 0x4B455947454E
plain = G.plain_mas(471)
table = cc.BigramTable(G.english_scores())
perm = np.random.default_rng(3).permutation(26)
cipher = perm[plain]
cfg = cc.MasSolverConfig(workers=64, climbings=10_000, restarts=20, global_seed=7000)
stop = lambda r: True  # noqa: E731  (stop after the first restart)
print("MAS solve_with_restarts (1 restart): min %.3f ms, median %.3f ms"
      % best_of(lambda: cc.solve_with_restarts(cipher, table, cfg, stop=stop)))
keys = philox_keys([7000] * 64, list(range(64)))
cof = np.zeros(64, np.int32)
print("MAS engine.mas_climb (64 x 10k): min %.3f ms, median %.3f ms"
      % best_of(lambda: engine.mas_climb([cipher], cof, keys, table.scores, 10_000)))
print("MAS engine.mas_climb (64 x 1): min %.3f ms, median %.3f ms"
      % best_of(lambda: engine.mas_climb([cipher], cof, keys, table.scores, 1)))
plain = G.plain_sct(596)
logs = cc.LogBigramTable(G.english_logs(), -24.0)
sc = cc.sct_encrypt(plain, np.random.default_rng(5).permutation(10))
scfg = cc.SctSolverConfig(key_length=10, workers=64, climbings=15_000, restarts=5, global_seed=8000)
print("SCT solve_sct (1 restart): min %.3f ms, median %.3f ms"
      % best_of(lambda: cc.solve_sct(sc, logs, scfg, stop=stop), 10))
print("SCT engine.sct_climb (64 x 15k): min %.3f ms, median %.3f ms"
      % best_of(lambda: engine.sct_climb([sc], cof, keys, logs.logs, 10, 15_000), 10))
print("SCT engine.sct_climb (64 x 1): min %.3f ms, median %.3f ms"
      % best_of(lambda: engine.sct_climb([sc], cof, keys, logs.logs, 10, 1), 10))
