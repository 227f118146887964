#!/usr/bin/env python
"""One MAS n-gram climb launch (for ncu): C4-like (125 ciphertexts of 60-100 letters from the
held-out sample, quadgram uint16 table) or --len L for fixed-length texts; prints evals/s."""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=4)
ap.add_argument("--len", type=int, default=0)
ap.add_argument("--restarts", type=int, default=1000)
ap.add_argument("--climbings", type=int, default=10_000)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
corpus = "".join(chr(97 + int(x)) for x in G.corpus())
q = cc.quantize_log_table(cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus, a.order)))
held = np.concatenate([G.plain_mas(637), G.plain_sct(596)])
rng = np.random.default_rng(4)
lengths = [a.len] * 125 if a.len else rng.integers(60, 101, 125)
ciphers = []
for i, L in enumerate(lengths):
    off = int(rng.integers(0, held.size - L))
    ciphers.append(rng.permutation(26)[held[off:off + L]])
cof = np.repeat(np.arange(125, dtype=np.int32), a.restarts)
keys = philox_keys([4000], list(range(cof.size)))
for r in range(a.reps):
    t0 = time.perf_counter()
    engine.mas_climb(ciphers, cof, keys, q.scores, a.climbings, order=a.order, group_size=a.restarts)
    dt = time.perf_counter() - t0
    print(f"order {a.order}: {cof.size * a.climbings / dt:.4g} evals/s ({dt:.3f} s)")
