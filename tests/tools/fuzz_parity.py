#!/usr/bin/env python
"""Randomized parity sweep of every GPU kernel against the CPU oracle for a time budget.

usage: python tests/tools/fuzz_parity.py [--seconds 300] [--seed 0]

Each round draws random inputs (text lengths, alphabets, tables across magnitudes and kernel
gates, budgets, stream keys, SCT key lengths / operator mixes, n-gram orders, deterministic
pivots) and compares per-worker outputs bit-for-bit with oracle/cc_oracle.c.  Prints one JSON
line with the counts per path; any mismatch raises with the failing case's parameters.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_2103_13937_b200 import engine  # noqa: E402
from paper_2103_13937_b200.rng import philox_keys  # noqa: E402


def texts(rng, n, lens):
    return [rng.integers(0, int(rng.integers(2, 27)), int(rng.choice(lens))) for _ in range(n)]


def fuzz_mas(rng, stats):
    tmax = int(rng.choice([1, 30, 700, 32_767, 65_535, 2**20, 2**33]))
    table = rng.integers(0, tmax + 1, 676)
    cs = texts(rng, 40, [2, 3, 7, 50, 200, 471, 1200, 5000])
    n = 400
    cof = rng.integers(0, len(cs), n).astype(np.int32)
    seeds, streams = rng.integers(0, 2**63, n).tolist(), rng.integers(0, 2**63, n).tolist()
    climb = int(rng.choice([1, 2, 17, 500, 2000, 6000]))
    kern = str(rng.choice(["auto", "dform", "dtable", "tform", "packed"]))
    res = engine.mas_climb(cs, cof, philox_keys(seeds, streams), table, climb, kernel=kern)
    s, m = O.mas_workers(cs, cof, seeds, streams, table, climb)
    if res.scores.tolist() != s.tolist() or not np.array_equal(res.keys.astype(np.int64), m):
        raise AssertionError(f"MAS mismatch: tmax={tmax} climb={climb} kernel={kern}")
    stats["mas_workers"] += n
    stats["mas_tries"] += n * climb


def fuzz_ngram(rng, stats):
    order = int(rng.choice([2, 3, 4]))
    table = rng.integers(0, int(rng.choice([2, 100, 65_536])), 26**order)
    cs = texts(rng, 30, [1, 2, 4, 30, 90, 300, 900])
    n = 200
    cof = rng.integers(0, len(cs), n).astype(np.int32)
    seeds, streams = rng.integers(0, 2**63, n).tolist(), rng.integers(0, 2**63, n).tolist()
    climb = int(rng.choice([1, 5, 300, 1500]))
    res = engine.mas_climb(cs, cof, philox_keys(seeds, streams), table, climb, order=order,
                           ngram_kernel=True)
    s, _ = O.ngram_workers(cs, cof, seeds, streams, order, table, climb)
    if res.scores.tolist() != s.tolist():
        raise AssertionError(f"n-gram mismatch: order={order} climb={climb}")
    stats["ngram_workers"] += n


def fuzz_sct(rng, stats):
    order = int(rng.choice([2, 2, 3, 4]))
    # kernel: speculative CTA / one warp per worker (one text length) or one worker per lane
    # (any mix of lengths)
    kernel = str(rng.choice(["warp", "warp", "lane"]))
    lens = [6, 64, 129, 400, 777]
    if kernel == "lane":
        cs = [rng.integers(0, 26, int(rng.choice(lens))) for _ in range(3)]
    else:
        n_len = int(rng.choice(lens))
        cs = [rng.integers(0, 26, n_len) for _ in range(3)]
    logs = -rng.random(26**order) * 20 - 1
    m = int(rng.choice([48, 80]))
    cof = rng.integers(0, 3, m).astype(np.int32)
    kmax = int(rng.choice([8, 20, 32, 64]))  # <= 32: narrow kernel variants
    klens = np.array([int(rng.integers(2, min(cs[c].size, kmax) + 1)) for c in cof], np.int32)
    seeds, streams = rng.integers(0, 2**63, m).tolist(), rng.integers(0, 2**63, m).tolist()
    p1, p2 = sorted(int(v) for v in rng.integers(0, 101, 2))
    hmax = 4 if kernel == "lane" else 10  # the lane kernels take up to 3 hops
    h1, h2 = int(rng.integers(1, hmax)), int(rng.integers(1, hmax))
    climb = int(rng.choice([0, 1, 50, 400, 3000]))
    # few workers: the chain-parsed speculative CTA kernel (hops <= 3), the replaying one, or
    # one warp per worker
    spec = [True, "replay", False][int(rng.integers(0, 3))]
    res = engine.sct_climb(cs, cof, philox_keys(seeds, streams), logs, klens, climb, p1=p1, p2=p2,
                           op1_hop=h1, op2_hop=h2, order=order, speculate=spec, kernel=kernel)
    for i in range(m):
        k = int(klens[i])
        key, score, _ = O.sct_worker(cs[cof[i]], logs, k, climb, seeds[i], streams[i], p1=p1,
                                     p2=p2, op1_hop=h1, op2_hop=h2, order=order)
        if float(res.scores[i]) != score or not np.array_equal(res.keys[i, :k].astype(np.int64), key):
            raise AssertionError(f"SCT mismatch: kernel={kernel} order={order} k={k} climb={climb}")
    stats["sct_workers"] += m
    stats["sct_lane_workers" if kernel == "lane" else "sct_warp_workers"] += m
    if kernel == "warp" and spec is True and max(h1, h2) <= 3:
        stats["sct_chain_workers"] += m


def fuzz_sct_fast(rng, stats):
    """The opt-in fast SCT mode (quantised, incremental) vs its full-rescore oracle."""
    import paper_2103_13937_b200 as cc

    order = int(rng.choice([2, 3, 4]))
    logs = -rng.random(26**order) * float(rng.choice([2, 20])) - 1
    lt = cc.LogNgramTable(order, logs, -30.0) if order > 2 else cc.LogBigramTable(logs, -30.0)
    q = cc.quantize_sct_table(lt, text_len=1000, max_shift=int(rng.choice([4, 10, 16])))
    cs = [rng.integers(0, int(rng.choice([3, 26])), int(rng.choice([5, 64, 129, 400, 1000])))
          for _ in range(3)]
    m = 64
    cof = rng.integers(0, 3, m).astype(np.int32)
    kmax = int(rng.choice([8, 20, 64]))
    klens = np.array([int(rng.integers(2, min(cs[c].size, kmax) + 1)) for c in cof], np.int32)
    seeds, streams = rng.integers(0, 2**63, m).tolist(), rng.integers(0, 2**63, m).tolist()
    p1, p2 = sorted(int(v) for v in rng.integers(0, 101, 2))
    h1, h2 = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    climb = int(rng.choice([0, 1, 60, 400]))
    res = engine.sct_fast_climb(cs, cof, philox_keys(seeds, streams), q, klens, climb, p1=p1,
                                p2=p2, op1_hop=h1, op2_hop=h2)
    for i in range(m):
        k = int(klens[i])
        key, score, _ = O.sct_fast_worker(cs[cof[i]], q.table, order, k, climb, seeds[i],
                                          streams[i], p1=p1, p2=p2, op1_hop=h1, op2_hop=h2)
        if int(res.scores[i]) != score or not np.array_equal(res.keys[i, :k].astype(np.int64), key):
            raise AssertionError(f"SCT fast mismatch: order={order} k={k} climb={climb}")
    stats["sct_fast_workers"] += m


def fuzz_det(rng, stats):
    table = rng.integers(0, int(rng.choice([3, 900, 2**31])), 676)
    cs = texts(rng, 12, [2, 5, 40, 300, 900])
    for c in cs:
        if np.unique(c).size < 2:
            c[0], c[-1] = 0, 1
    iters = int(rng.choice([1, 20, 120]))
    seed = int(rng.integers(0, 2**63))
    keys = philox_keys([seed], [((r << 32) | (2**32 - 1)) for r in range(len(cs))])
    res = engine.mas_det_solve(cs, np.arange(len(cs), dtype=np.int32), keys, table, iters)
    for r, c in enumerate(cs):
        t, s, h = O.solve_deterministic(c, table, iters, seed, r)
        if int(res.scores[r]) != s or res.history[r] != h:
            raise AssertionError(f"deterministic mismatch: iters={iters}")
    stats["det_jobs"] += len(cs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    stats = {"rounds": 0, "mas_workers": 0, "mas_tries": 0, "ngram_workers": 0, "sct_workers": 0,
             "sct_warp_workers": 0, "sct_lane_workers": 0, "sct_chain_workers": 0, "sct_fast_workers": 0, "det_jobs": 0}
    t0 = time.time()
    while time.time() - t0 < a.seconds:
        for f in (fuzz_mas, fuzz_ngram, fuzz_sct, fuzz_sct_fast, fuzz_det):
            f(rng, stats)
        stats["rounds"] += 1
    stats["seconds"] = round(time.time() - t0, 1)
    stats["mismatches"] = 0
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
