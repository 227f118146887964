#!/usr/bin/env python
"""Small runs of every climb kernel for compute-sanitizer (memcheck / racecheck / synccheck):
D-form / T-form / packed MAS, n-gram orders 2-4 (with the table-read counter), deterministic
MAS, SCT warp / speculative / per-lane kernels (ragged text lengths, orders 2-4) and the fast
SCT mode; the L2 / smem microbenchmarks.  Checks results against the oracle as well."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_2103_13937_b200 import engine  # noqa: E402
from paper_2103_13937_b200.rng import philox_keys  # noqa: E402

rng = np.random.default_rng(5)
cs = [rng.integers(0, 26, int(L)) for L in (40, 97, 300)]
cof = np.array([0, 1, 2, 2, 1, 0, 2, 1], np.int32)
seeds, streams = [3] * 8, list(range(8))
keys = philox_keys(seeds, streams)
table = rng.integers(0, 700, 676)
for kern in ("dform", "dtable", "tform", "packed"):
    r = engine.mas_climb(cs, cof, keys, table, 300, kernel=kern)
    s, _ = O.mas_workers(cs, cof, seeds, streams, table, 300)
    assert r.scores.tolist() == s.tolist(), kern
for order in (2, 3, 4):
    t = rng.integers(0, 60000, 26**order)
    r = engine.mas_climb(cs, cof, keys, t, 300, order=order, ngram_kernel=True)
    s, _ = O.ngram_workers(cs, cof, seeds, streams, order, t, 300)
    assert r.scores.tolist() == s.tolist(), order
dk = philox_keys([9], [(r << 32) | (2**32 - 1) for r in range(3)])
d = engine.mas_det_solve(cs, np.arange(3, dtype=np.int32), dk, table, 20)
for j, c in enumerate(cs):
    _, sc, _ = O.solve_deterministic(c, table, 20, 9, j)
    assert int(d.scores[j]) == sc
logs = -rng.random(676) * 20 - 1
sc_c = [rng.integers(0, 26, 200) for _ in range(2)]
sc_cof = np.array([0, 1, 1, 0], np.int32)
sk = philox_keys([4] * 4, list(range(4)))
# latency kernels: two SMs per worker (4 workers), the replaying CTA kernel, one warp
for spec in (True, "replay", False):
    r = engine.sct_climb(sc_c, sc_cof, sk, logs, 9, 60, speculate=spec)
    for i in range(4):
        _, s, _ = O.sct_worker(sc_c[sc_cof[i]], logs, 9, 60, 4, i)
        assert float(r.scores[i]) == s, (spec, i)
# the one-CTA chain kernel (more workers than SM pairs), a climb spanning parse chunks
ch_cof = (np.arange(80) % 2).astype(np.int32)
ch_k = philox_keys([5] * 80, list(range(80)))
r = engine.sct_climb(sc_c, ch_cof, ch_k, logs, 9, 700)
for i in (0, 1, 79):
    _, s, _ = O.sct_worker(sc_c[ch_cof[i]], logs, 9, 700, 5, i)
    assert float(r.scores[i]) == s, ("chain", i)
# per-lane SCT kernels: parity (orders 2-4, ragged lengths, a chunk spanning ciphertexts) and
# the fast mode
lane_c = [rng.integers(0, 26, int(L)) for L in (200, 57, 333)]
lane_cof = np.array([0] * 20 + [1, 2] * 10 + [2] * 5, np.int32)
lane_k = np.array([int(rng.integers(2, 12)) for _ in lane_cof], np.int32)
lane_keys = philox_keys([6] * lane_cof.size, list(range(lane_cof.size)))
for order in (2, 3, 4):
    lg = -rng.random(26**order) * 20 - 1
    r = engine.sct_climb(lane_c, lane_cof, lane_keys, lg, lane_k, 40, order=order, kernel="lane")
    for i in (0, 21, 44):
        _, s, _ = O.sct_worker(lane_c[lane_cof[i]], lg, int(lane_k[i]), 40, 6, i, order=order)
        assert float(r.scores[i]) == s, (order, i)
    import paper_2103_13937_b200 as cc  # noqa: E402
    lt = cc.LogNgramTable(order, lg, -30.0) if order > 2 else cc.LogBigramTable(lg, -30.0)
    q = cc.quantize_sct_table(lt, text_len=400)
    r = engine.sct_fast_climb(lane_c, lane_cof, lane_keys, q, lane_k, 40)
    for i in (0, 21, 44):
        _, s, _ = O.sct_fast_worker(lane_c[lane_cof[i]], q.table, order, int(lane_k[i]), 40, 6, i)
        assert int(r.scores[i]) == s, (order, i)
    # regular grids (every k divides 200): the window-sum tables (sct_ftab_kernel)
    reg_cof = np.zeros(40, np.int32)
    reg_k = np.array([(4, 5, 8, 10)[i % 4] for i in range(40)], np.int32)
    r = engine.sct_fast_climb(lane_c, reg_cof, lane_keys[:40], q, reg_k, 40)
    for i in (0, 1, 2, 3):
        _, s, _ = O.sct_fast_worker(lane_c[0], q.table, order, int(reg_k[i]), 40, 6, i)
        assert int(r.scores[i]) == s, ("regular", order, i)
t4 =rng.integers(0, 60000, 26**4)
engine.mas_climb(cs, cof, keys, t4, 200, order=4, computed=True, lookups=True)
engine.bench_l2_gather(26**4)
# scoring / delta / test-set kernels
from paper_2103_13937_b200 import ciphers as C  # noqa: E402
from paper_2103_13937_b200 import rng as R  # noqa: E402
texts = [rng.integers(0, 26, int(L)) for L in (0, 1, 2, 9, 130, 600)]
for order in (2, 3, 4):
    t = rng.integers(0, 1000, 26**order)
    got = engine.ngram_score_batch(texts, order, t)
    assert got.tolist() == [int(O.ngram_score_text(x, order, t)) for x in texts], order
    lg = -rng.random(26**order) * 10 - 1
    got = engine.ngram_log_score_batch(texts, order, lg)
    assert got.tolist() == [O.ngram_log_score_text(x, order, lg) for x in texts], order
pairs = np.array([[0, 1], [3, 7], [25, 24]], np.int32)
engine.mas_delta_batch(texts[3:], pairs, table)
keys10 = np.array([rng.permutation(9) for _ in range(4)], np.uint8)
engine.sct_score_batch(sc_c, sc_cof, keys10, logs)
C.encrypt_batch([rng.integers(0, 26, 50) for _ in range(5)], "mas", key_seeds=list(range(5)))
C.encrypt_batch([rng.integers(0, 26, 50) for _ in range(5)], "sct", key_seeds=list(range(5)),
                key_lengths=[5, 6, 7, 8, 9])
R.draws(5, 7, 300)
print("sanitize smoke ok")
