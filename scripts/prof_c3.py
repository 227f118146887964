#!/usr/bin/env python
"""One C3-shaped SCT launch for ncu: 1,000 ciphertexts x 400 letters, k = 5..20 (ragged),
trigram log table, 64 workers each, --climbings tries (default 1,000), --kernel auto / lane /
warp / fast."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "tests" / "tools"))
import bench_configs as BC  # noqa: E402
import paper_2103_13937_b200 as cc  # noqa: E402
from paper_2103_13937_b200 import engine  # noqa: E402
from paper_2103_13937_b200.rng import philox_keys  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--climbings", type=int, default=1000)
ap.add_argument("--kernel", default="auto")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--table-l2", action="store_true")
a = ap.parse_args()
l3 = cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(BC.corpus_text(), 3))
ciphers, plains, kofc = BC.c3_inputs()
W = 64
cof = np.repeat(np.arange(len(ciphers), dtype=np.int32), W)
klens = np.repeat(np.array(kofc, dtype=np.int32), W)
keys = philox_keys([9000], list(range(cof.size)))
q = cc.quantize_sct_table(l3, text_len=400) if a.kernel == "fast" else None
for _ in range(a.reps):
    t0 = time.perf_counter()
    if a.kernel == "fast":
        engine.sct_fast_climb(ciphers, cof, keys, q, klens, a.climbings, group_size=W,
                              table_l2=a.table_l2)
    else:
        engine.sct_climb(ciphers, cof, keys, l3.logs, klens, a.climbings, order=3, group_size=W,
                         kernel=a.kernel, table_l2=a.table_l2)
    dt = time.perf_counter() - t0
    print(f"C3 {a.kernel}{' table_l2' if a.table_l2 else ''}: {cof.size * a.climbings / dt:.4g} "
          f"evals/s ({dt:.3f} s)")
