#!/usr/bin/env python
"""One warm-up launch (100 climbings) then one SCT restart of the acceptance #08 shape on the
default latency kernel -- for ncu with SKIP=1."""
import sys
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
spec = {"chain": True, "replay": "replay", "warp": False}[sys.argv[2] if len(sys.argv) > 2 else "chain"]
plain = G.plain_sct(596)
logs = cc.LogBigramTable(G.english_logs(), -24.0).logs
cipher = cc.sct_encrypt(plain, np.random.default_rng(5).permutation(k))
keys = philox_keys([8000], list(range(64)))
cof = np.zeros(64, np.int32)
engine.sct_climb([cipher], cof, keys, logs, k, 100, speculate=spec)
r = engine.sct_climb([cipher], cof, keys, logs, k, 15_000, speculate=spec, last_accept=True)
print("accepted-by (last accept per worker, median):", int(np.median(r.last_accept)))
