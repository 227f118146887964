#!/usr/bin/env python
"""One SCT restart of the acceptance #08 shape (64 workers x 15,000 climbings, 596 letters) on
each latency-mode kernel: the chain-parsed one (default), the per-round replay one, and one
warp per worker; outputs must agree."""
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

plain = G.plain_sct(596)
logs = cc.LogBigramTable(G.english_logs(), -24.0).logs
for k in (int(x) for x in (sys.argv[1:] or ["10", "15"])):
    cipher = cc.sct_encrypt(plain, np.random.default_rng(5).permutation(k))
    keys = philox_keys([8000], list(range(64)))
    cof = np.zeros(64, np.int32)
    res = {}
    for name, spec in (("chain", True), ("replay", "replay"), ("warp", False)):
        engine.sct_climb([cipher], cof, keys, logs, k, 100, speculate=spec)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = engine.sct_climb([cipher], cof, keys, logs, k, 15_000, speculate=spec,
                                 draws_used=True)
            ts.append(time.perf_counter() - t0)
        res[name] = r
        print(f"k={k} {name}: one restart (64 x 15000) {1e3 * min(ts):.2f} ms; "
              f"{1e6 * min(ts) / 15000:.3f} us/try", flush=True)
    for name in ("chain", "replay"):
        same = (res[name].scores.tolist() == res["warp"].scores.tolist()
                and np.array_equal(res[name].keys, res["warp"].keys)
                and np.array_equal(res[name].draws_used, res["warp"].draws_used))
        print(f"k={k} {name} identical to warp: {same}")
