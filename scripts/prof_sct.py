#!/usr/bin/env python
"""One SCT climb launch at full occupancy (for ncu): k=10, n=400, bigram (or --order 3),
--workers workers x --climbings climbings; prints evals/s measured around the engine call."""
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
ap.add_argument("--order", type=int, default=2)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--workers", type=int, default=16384)
ap.add_argument("--climbings", type=int, default=2000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kernel", default="auto", help="auto / lane / warp / fast")
a = ap.parse_args()
corpus = "".join(chr(97 + int(x)) for x in G.corpus())
if a.order == 2:
    logs = G.english_logs()
else:
    logs = cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus, a.order)).logs
plain = G.plain_sct(400)
cipher = cc.sct_encrypt(plain, np.random.default_rng(3).permutation(a.k))
keys = philox_keys([11], list(range(a.workers)))
cof = np.zeros(a.workers, np.int32)
if a.kernel == "fast":
    lt = cc.LogNgramTable(a.order, logs, float(np.min(logs))) if a.order > 2 else \
        cc.LogBigramTable(logs, -24.0)
    q = cc.quantize_sct_table(lt, text_len=400)
for r in range(a.reps):
    t0 = time.perf_counter()
    if a.kernel == "fast":
        res = engine.sct_fast_climb([cipher], cof, keys, q, a.k, a.climbings)
    else:
        res = engine.sct_climb([cipher], cof, keys, logs, a.k, a.climbings, order=a.order,
                               kernel=a.kernel)
    dt = time.perf_counter() - t0
    extra = ""
    if res.lookups is not None:
        extra = f", {res.lookups.sum() / (a.workers * a.climbings):.1f} lookups/eval"
    print(f"{a.kernel} order {a.order} k {a.k}: {a.workers * a.climbings / dt:.4g} evals/s "
          f"({dt:.3f} s{extra})")
