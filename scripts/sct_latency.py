#!/usr/bin/env python
"""Latency of one SCT restart (64 workers x 15,000 climbings, k=10, 596 letters -- the
acceptance #08 shape) through engine.sct_climb: the time-to-recover building block, bound by
one worker's sequential tries rather than by throughput."""
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

k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
plain = G.plain_sct(596)
cipher = cc.sct_encrypt(plain, np.random.default_rng(5).permutation(k))
logs = cc.LogBigramTable(G.english_logs(), -24.0).logs
keys = philox_keys([8000], list(range(64)))
cof = np.zeros(64, np.int32)
engine.sct_climb([cipher], cof, keys, logs, k, 100)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    engine.sct_climb([cipher], cof, keys, logs, k, 15_000)
    ts.append(time.perf_counter() - t0)
print(f"k={k}: one restart (64 x 15000) {1e3 * min(ts):.1f} ms; {1e6 * min(ts) / 15000:.2f} us/try")
