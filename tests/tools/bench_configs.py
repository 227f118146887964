#!/usr/bin/env python
"""Throughput, time-to-recover and parity on BASELINE.json's other configurations
(bench.py's headline is configs[1] = C2; bench.py also embeds run_all(bounded=True) as the
"configs" block of its JSON line, so the driver's own run records these numbers).

  C1  MAS, one 300-letter held-out ciphertext (acceptance #07 recipe, key_seed 700), bigram,
      64 workers x 10,000 climbings x R restarts.
  C1d the deterministic best-neighbour solver on the same ciphertext (mas.py:140-169),
      R restarts x 500 iterations x 325 candidates.
  C3  SCT, key lengths 5..20, 1,000 ciphertexts of 400 letters, trigram log table (parity
      mode: float64, numpy pairwise order) -- and the opt-in quantised incremental mode
      (engine.sct_fast_climb) with its key agreement against the parity mode.
  C4  MAS, 60-100 letter ciphertexts, quadgram (uint16 quantised log table, read via L2),
      one worker per restart.
  C5  evals/s vs workers and n-gram order 2/3/4.
  TTR time to recover the key on the reference's acceptance recipes #07 (MAS) and #08 (SCT)
      (tests/test_acceptance.py:146-198), stop on the plaintext, public API.

Every timed call goes through the public engine API from host buffers (H2D + D2H inside the
timed region) after a warm-up call; evals count executed fitness evaluations only.  The CPU
numbers are the C oracle (oracle/cc_oracle.c, a port of the reference algorithm -- test
infrastructure, used here only as the CPU baseline and the parity checker) on all host
cores over a bounded sample of the same work; each entry's "parity" compares a sample of
the GPU's per-worker outputs with the oracle's bit for bit.

usage: python tests/tools/bench_configs.py [--quick] [--only C1,C3,...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
for p in (ROOT, ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

import golden_data as G  # noqa: E402
import paper_2103_13937_b200 as cc  # noqa: E402
from paper_2103_13937_b200 import engine  # noqa: E402
from paper_2103_13937_b200.rng import philox_keys  # noqa: E402

KEYGEN = 2**32 - 2
THREADS = os.cpu_count() or 1



C3_PROFILE = "profiles/r2h_c3_lane_ncu.txt"


def _ncu_counter(rel, pat):
    """One counter from a committed profiles/*_ncu.txt summary (None if absent)."""
    import re

    try:
        txt = (Path(__file__).resolve().parents[2] / rel).read_text()
    except OSError:
        return None
    m = re.search(pat + r"\s+([0-9.eE+]+)", txt)
    return float(m.group(1)) if m else None


def timed(fn, reps=1):
    fn()  # warm-up (also loads tables / allocates scratch)
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    return out, (time.perf_counter() - t0) / reps


def corpus_text():
    return "".join(chr(97 + int(x)) for x in G.corpus())


def cpu_rate(fn, evals_of, budget_s=4.0):
    """Run fn(m) for growing m until it takes >= budget_s; return (evals/s, m)."""
    m = 1
    while True:
        t0 = time.perf_counter()
        fn(m)
        dt = time.perf_counter() - t0
        if dt >= budget_s or m >= 1 << 20:
            return evals_of(m) / dt, m
        m = max(m + 1, int(m * min(8.0, 1.5 * budget_s / max(dt, 1e-3))))


def _c1_input():
    from oracle import oracle as O

    plain = G.plain_mas(300)
    cipher = O.permutation(700, KEYGEN, 26)[plain]
    return plain, cipher, cc.BigramTable(G.english_scores())


def c1(bounded=False, quick=False):
    from oracle import oracle as O

    plain, cipher, table = _c1_input()
    R = 2000 if (quick or bounded) else 10_000
    W, K = 64, 10_000
    streams = [(r << 32) | w for r in range(R) for w in range(W)]
    keys = philox_keys([7000], streams)
    res, dt = timed(lambda: engine.mas_climb([cipher], np.zeros(len(streams), np.int32), keys,
                                             table.scores, K, group_size=W))
    evals = len(streams) * K
    best = int(np.argmax(res.scores))
    rate_cpu, m = cpu_rate(lambda m: O.mas_workers([cipher], np.zeros(m * THREADS, np.int32),
                                                   [7000] * (m * THREADS), streams[:m * THREADS],
                                                   table.scores, K, threads=THREADS),
                           lambda m: m * THREADS * K, budget_s=2.0 if bounded else 4.0)
    # parity: restarts 0 and R-1, every worker, against the oracle
    idx = list(range(W)) + list(range((R - 1) * W, R * W))
    ws, wm = O.mas_workers([cipher], np.zeros(len(idx), np.int32), [7000] * len(idx),
                           [streams[i] for i in idx], table.scores, K, threads=THREADS)
    exact = bool(np.array_equal(ws, res.scores[idx])
                 and np.array_equal(wm, res.keys[idx].astype(np.int64)))
    true_score = int(cc.score_text(plain, table))
    return {"config": "C1", "what": "MAS n=300 bigram, 64 workers x 10k climbings x restarts",
            "restarts": R, "evals": evals, "seconds": dt, "evals_per_s": evals / dt,
            "cpu_evals_per_s": rate_cpu, "cpu_cores": THREADS, "cpu_kind": "port",
            "parity": {"bit_exact": exact, "sample": f"{len(idx)} workers (restarts 0 and "
                                                      f"{R - 1}): scores and letter maps"},
            "best_score": int(res.scores[best]), "true_plaintext_score": true_score,
            "restarts_recovering_plaintext": int(sum(
                np.array_equal(res.keys[r * W + int(res.group_best[r])].astype(np.int64)[cipher],
                               plain) for r in range(R))),
            "note": "the best fitness found exceeds the true plaintext's with the reference's "
                    "17.5k-letter bigram table (SURVEY A14): no search recovers this key"}


def c1d(bounded=False, quick=False):
    from oracle import oracle as O

    plain, cipher, table = _c1_input()
    R = 2000 if (quick or bounded) else 20_000
    keys = philox_keys([606], [(r << 32) | (2**32 - 1) for r in range(R)])
    res, dt = timed(lambda: engine.mas_det_solve([cipher], np.zeros(R, np.int32), keys,
                                                 table.scores, 500))
    evals = R * 500 * 325
    rate_cpu, m = cpu_rate(lambda m: [O.solve_deterministic(cipher, table.scores, 500, 606, r)
                                      for r in range(m)], lambda m: m * 500 * 325,
                           budget_s=1.5 if bounded else 3.0)
    exact = all(O.solve_deterministic(cipher, table.scores, 500, 606, r)[1] == int(res.scores[r])
                for r in range(3))
    return {"config": "C1d", "what": "deterministic best-neighbour MAS n=300, 500 iterations "
                                     "x 325 candidates per restart", "restarts": R,
            "evals": evals, "seconds": dt, "evals_per_s": evals / dt,
            "cpu_evals_per_s": rate_cpu, "cpu_cores": 1, "cpu_kind": "port",
            "parity": {"bit_exact": bool(exact), "sample": "restarts 0-2: final scores"},
            "best_score": int(res.scores.max())}


def c3_inputs():
    from oracle import oracle as O

    corpus = G.corpus()
    ciphers, plains, kofc = [], [], []
    for i in range(1000):
        k = 5 + i % 16
        off = int(np.random.default_rng(300000 + i).integers(0, corpus.size - 400))
        p = corpus[off:off + 400]
        key = O.permutation(300000 + i, KEYGEN, k)
        plains.append(p)
        ciphers.append(cc.sct_encrypt(p, key))
        kofc.append(k)
    return ciphers, plains, kofc


def _recovered(ciphers, plains, kofc, res, W, idx=None):
    idx = range(len(ciphers)) if idx is None else idx
    return [bool(np.array_equal(cc.sct_decrypt(ciphers[j], res.keys[j * W + int(res.group_best[j]),
                                                                    :kofc[j]].astype(np.int64)),
                                plains[j])) for j in idx]


def c3(bounded=False, quick=False):
    from oracle import oracle as O

    l3 = cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus_text(), 3))
    ciphers, plains, kofc = c3_inputs()
    n_c = len(ciphers)
    W, K = (8, 1000) if quick else (64, 15_000)  # SctSolverConfig defaults (sct.py:47-48)
    cof = np.repeat(np.arange(n_c, dtype=np.int32), W)
    klens = np.repeat(np.array(kofc, dtype=np.int32), W)
    keys = philox_keys([9000], list(range(cof.size)))
    res, total_s = timed(lambda: engine.sct_climb(ciphers, cof, keys, l3.logs, klens, K, order=3,
                                                  group_size=W))
    total_evals = cof.size * K
    rec = _recovered(ciphers, plains, kofc, res, W)
    rows = []
    for k in range(5, 21):
        idx = [j for j in range(n_c) if kofc[j] == k]
        rows.append({"k": k, "ciphers": len(idx), "recovered": int(sum(rec[j] for j in idx))})
    # parity: every worker of one ciphertext per key length (16 x W workers) vs the oracle
    exact = True
    for k in range(5, 21):
        j = k - 5
        ws, wk = O.sct_workers([ciphers[j]], np.zeros(W, np.int32), [9000] * W,
                               list(range(j * W, (j + 1) * W)), l3.logs, k, K, order=3,
                               threads=THREADS)
        exact &= bool(np.array_equal(ws, res.scores[j * W:(j + 1) * W])
                      and np.array_equal(wk, res.keys[j * W:(j + 1) * W, :k].astype(np.int64)))
    c0 = ciphers[15]
    rate_cpu, m = cpu_rate(lambda m: O.sct_workers([c0], np.zeros(m * THREADS, np.int32),
                                                   [9000] * (m * THREADS), list(range(m * THREADS)),
                                                   l3.logs, 20, 200, order=3, threads=THREADS),
                           lambda m: m * THREADS * 200, budget_s=2.0 if bounded else 4.0)
    # the SCT climb reads, per evaluation, every plaintext letter through the column starts
    # (n shared-memory gathers) and every window's table entry (n - 2 gathers): the
    # reference algorithm's O(n) lookups, against the LDS lane-lookup peak
    lpe = 400 + 398
    peak = 148 * 32 * 1.965e9
    roof = {"bound": "smem-lookups", "lookups_per_eval": lpe,
            "achieved": total_evals / total_s * lpe, "peak": peak, "unit": "lookups/s",
            "frac": total_evals / total_s * lpe / peak,
            "peak_source": "148 SMs x 32 lane lookups per clock x 1965 MHz (SURVEY 8d formula)"}
    # the counter-based bound: shared-memory wavefronts per evaluation from the committed ncu
    # capture of the same launch shape (1,000 climbings) x this run's rate, against one
    # wavefront per SM per clock -- the random text / table gathers replay on bank conflicts,
    # so this, not the lane-lookup peak, is the pipe the kernel fills
    wf = _ncu_counter(C3_PROFILE, r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum")
    tr = _ncu_counter(C3_PROFILE, r"tries in the captured launch:")
    pipe = None
    if wf and tr:
        wpe = wf / tr
        wpeak = 148 * 1.965e9
        pipe = {"bound": "smem-pipe", "wavefronts_per_eval": wpe,
                "achieved": total_evals / total_s * wpe, "peak": wpeak, "unit": "wavefronts/s",
                "frac": total_evals / total_s * wpe / wpeak,
                "ncu_pct_of_peak": _ncu_counter(C3_PROFILE, r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum\.pct_of_peak_sustained_elapsed"),
                "source": f"ncu wavefronts / tries ({C3_PROFILE}) x this run's evals/s; peak = 1 "
                          "wavefront per SM per clock at 1965 MHz"}
    out = [{"config": "C3", "what": "SCT k=5..20, 1000 ciphertexts x 400 letters, trigram log "
                                    "table, parity mode (float64, numpy pairwise order)",
            "roofline": roof, "smem_pipe_roofline": pipe,
            "workers_per_cipher": W, "climbings": K, "launches": "one (ragged key lengths)",
            "evals": total_evals, "seconds": total_s, "evals_per_s": total_evals / total_s,
            "recovered": int(sum(rec)), "of": n_c,
            "cpu_evals_per_s": rate_cpu, "cpu_cores": THREADS, "cpu_kind": "port",
            "parity": {"bit_exact": bool(exact),
                       "sample": f"all {W} workers of one ciphertext per key length (k=5..20): "
                                 "float64 scores and keys"},
            "per_k": rows}]
    if hasattr(engine, "sct_fast_climb"):
        out.append(c3_fast(ciphers, plains, kofc, l3, W, K, res, rec, bounded))
    return out


def c3_fast(ciphers, plains, kofc, l3, W, K, res_parity, rec_parity, bounded=False):
    """The opt-in fast SCT mode on C3: quantised int32 table, incremental rescoring of the
    windows touching the columns a candidate moves (engine.sct_fast_climb); its own oracle
    (oracle.sct_fast_workers) pins it bit-exactly, and its final keys are compared with the
    parity mode's."""
    from oracle import oracle as O

    n_c = len(ciphers)
    q = cc.quantize_sct_table(l3, text_len=400)
    cof = np.repeat(np.arange(n_c, dtype=np.int32), W)
    klens = np.repeat(np.array(kofc, dtype=np.int32), W)
    keys = philox_keys([9000], list(range(cof.size)))
    res, dt = timed(lambda: engine.sct_fast_climb(ciphers, cof, keys, q, klens, K,
                                                  group_size=W))
    evals = cof.size * K
    same_worker = float(np.mean([np.array_equal(res.keys[i, :klens[i]],
                                                 res_parity.keys[i, :klens[i]])
                                 for i in range(cof.size)]))
    same_best = float(np.mean([np.array_equal(
        res.keys[j * W + int(res.group_best[j]), :kofc[j]],
        res_parity.keys[j * W + int(res_parity.group_best[j]), :kofc[j]]) for j in range(n_c)]))
    rec = _recovered(ciphers, plains, kofc, res, W)
    exact = True
    for k in (5, 13, 20):
        j = k - 5
        ws, wk = O.sct_fast_workers([ciphers[j]], np.zeros(W, np.int32), [9000] * W,
                                    list(range(j * W, (j + 1) * W)), q.table, 3, k, K,
                                    threads=THREADS)
        exact &= bool(np.array_equal(ws, res.scores[j * W:(j + 1) * W])
                      and np.array_equal(wk, res.keys[j * W:(j + 1) * W, :k].astype(np.int64)))
    looks = None if res.lookups is None else float(res.lookups.sum() / evals)
    return {"config": "C3-fast", "what": "SCT k=5..20, 1000 x 400 letters, trigram, opt-in fast "
                                         "mode: int32-quantised table (scale 2^%d), incremental "
                                         "rescoring of the windows of moved columns" % q.shift,
            "workers_per_cipher": W, "climbings": K, "evals": evals, "seconds": dt,
            "evals_per_s": evals / dt, "table_lookups_per_eval": looks,
            "recovered": int(sum(rec)), "recovered_parity_mode": int(sum(rec_parity)), "of": n_c,
            "agreement": {"final_key_per_worker": same_worker, "best_key_per_cipher": same_best,
                          "vs": "parity mode (float64 pairwise), same streams"},
            "parity": {"bit_exact": bool(exact),
                       "sample": "all workers of three ciphertexts (k=5, 13, 20) vs the fast "
                                 "mode's oracle (oracle/cc_oracle.c cco_sct_fast_worker)"}}


def c4(bounded=False, quick=False):
    from oracle import oracle as O

    q4 = cc.quantize_log_table(cc.build_log_ngram_table(
        cc.build_ngram_table_from_corpus(corpus_text(), 4)))
    n_c = 125
    R = 200 if quick else 1000
    K = 10_000
    held = np.concatenate([G.plain_mas(637), G.plain_sct(596)])
    lengths = np.random.default_rng(4).integers(60, 101, n_c)
    ciphers, plains = [], []
    for i, L in enumerate(lengths):
        off = int(np.random.default_rng(400000 + i).integers(0, held.size - L))
        p = held[off:off + L]
        plains.append(p)
        ciphers.append(O.permutation(400000 + i, KEYGEN, 26)[p])
    cof = np.repeat(np.arange(n_c, dtype=np.int32), R)
    keys = philox_keys([4000], list(range(cof.size)))
    res, dt = timed(lambda: engine.mas_climb(ciphers, cof, keys, q4.scores, K, order=4,
                                             group_size=R, computed=True, lookups=True))
    evals = cof.size * K
    ok = sum(np.array_equal(res.keys[j * R + int(res.group_best[j])].astype(np.int64)[ciphers[j]],
                            plains[j]) for j in range(n_c))
    rate_cpu, m = cpu_rate(lambda m: O.ngram_workers([ciphers[0]], np.zeros(m * THREADS, np.int32),
                                                     [4000] * (m * THREADS),
                                                     list(range(m * THREADS)), 4, q4.scores, 2000,
                                                     threads=THREADS),
                           lambda m: m * THREADS * 2000, budget_s=2.0 if bounded else 4.0)
    idx = list(range(256)) + list(range((n_c - 1) * R, (n_c - 1) * R + 256))
    ws, wm = O.ngram_workers([ciphers[0], ciphers[-1]], np.array([0] * 256 + [1] * 256, np.int32),
                             [4000] * 512, idx, 4, q4.scores, K, threads=THREADS)
    exact = bool(np.array_equal(ws, res.scores[idx])
                 and np.array_equal(wm, res.keys[idx].astype(np.int64)))
    walks = float(res.computed.sum() / evals)
    lpe = float(res.lookups.sum() / evals)
    peak = engine.bench_l2_gather(26**4)
    roof = {"bound": "l2-gather", "lookups_per_eval": lpe, "achieved": evals / dt * lpe,
            "peak": peak, "unit": "gathers/s", "frac": evals / dt * lpe / peak,
            "peak_source": "ccg_bench_l2_gather: random uint16 gathers from a 26^4-entry "
                           "(914 KB) table at full occupancy, measured in this run",
            "note": "quadgram table reads executed by the climb (position walks of cache "
                    "misses + window refreshes after accepts, counted on the device); the "
                    "wall time also includes the H2D/D2H of the public API call"}
    return {"config": "C4", "what": "MAS 60-100 letters, quadgram uint16 table via L2, one "
                                    "worker per restart", "ciphers": n_c,
            "restarts_per_cipher": R, "climbings": K, "evals": evals, "seconds": dt,
            "evals_per_s": evals / dt, "computed_by_walk": walks, "roofline": roof,
            "recovered": int(ok), "of": n_c, "cpu_evals_per_s": rate_cpu, "cpu_cores": THREADS,
            "cpu_kind": "port (full rescore per try)",
            "parity": {"bit_exact": exact, "sample": "512 workers (first 256 of the first and "
                                                     "last ciphertext): scores and letter maps"}}


def c5(bounded=False, quick=False):
    corpus = corpus_text()
    tabs = {2: cc.BigramTable(G.english_scores()).scores}
    for o in (3, 4):
        tabs[o] = cc.quantize_log_table(cc.build_log_ngram_table(
            cc.build_ngram_table_from_corpus(corpus, o))).scores
    plain = G.plain_mas(300)
    cipher = np.random.default_rng(1).permutation(26)[plain]
    K = 10_000
    if bounded:
        sizes = [1000, 100_000, 1_000_000]
    else:
        sizes = [1000, 10_000, 100_000] + ([] if quick else [1_000_000, 10_000_000])
    key_cache, lines = {}, []
    for order in (2, 3, 4):
        for n in sizes:
            if n not in key_cache:
                key_cache[n] = philox_keys([5], list(range(n)))
            keys = key_cache[n]
            res, dt = timed(lambda: engine.mas_climb([cipher], np.zeros(n, np.int32), keys,
                                                     tabs[order], K, order=order,
                                                     computed=order > 2))
            line = {"config": "C5", "order": order, "workers": n, "climbings": K,
                    "text_len": 300, "evals_per_s": n * K / dt, "seconds": dt}
            if order > 2:
                line["computed_by_walk"] = float(res.computed.sum() / (n * K))
            lines.append(line)
    return lines


def ttr(bounded=False, quick=False):
    """Time to recover the key on the reference's acceptance recipes (tests/test_acceptance.py
    :146-198; BASELINE.json metric "time-to-recover key"): MAS #07 (471 letters, 10 keys,
    64 workers x 10k, <= 20 restarts) and SCT #08 (596 letters, k = 10 / 15, 64 x 15k,
    <= 5 / 10 restarts), stop on the exact plaintext, through the public API.  CPU column:
    the C oracle port on all host cores running the same restarts until the same stop; the
    GPU's and the port's outcomes (recovered, restarts used) must agree key by key."""
    from oracle import oracle as O

    out = []
    plain = G.plain_mas(471)
    table = cc.BigramTable(G.english_scores())
    # warm-up (context, module load) outside the timed solves
    cc.solve_with_restarts(O.permutation(1, KEYGEN, 26)[plain], table,
                           cc.MasSolverConfig(workers=64, climbings=1000, restarts=2))
    gpu_t, cpu_t, ok, ok_cpu, restarts, restarts_cpu = [], [], 0, 0, [], []
    for e in range(3 if quick else 10):
        cipher = O.permutation(700 + e, KEYGEN, 26)[plain]
        cfg = cc.MasSolverConfig(workers=64, climbings=10_000, restarts=20, global_seed=7000 + e)
        t0 = time.perf_counter()
        best, summ = cc.solve_with_restarts(cipher, table, cfg,
                                            stop=lambda r: bool(np.array_equal(r.best_text, plain)))
        gpu_t.append(time.perf_counter() - t0)
        ok += bool(np.array_equal(best.best_text, plain))
        restarts.append(len(summ))
        t0 = time.perf_counter()
        used = 20
        for r in range(20):
            s, m = O.mas_workers([cipher], np.zeros(64, np.int32), [7000 + e] * 64,
                                 [(r << 32) | w for w in range(64)], table.scores, 10_000,
                                 threads=THREADS)
            if np.array_equal(m[int(np.argmax(s))][cipher], plain):
                ok_cpu += 1
                used = r + 1
                break
        restarts_cpu.append(used)
        cpu_t.append(time.perf_counter() - t0)
    out.append({"config": "TTR-07", "what": "acceptance #07 MAS: 10 keys, 471 letters, 64 x "
                                            "10k, <= 20 restarts, stop on the plaintext",
                "recovered": ok, "of": len(gpu_t), "restarts_used": restarts,
                "gpu_ms_per_key": 1e3 * sum(gpu_t) / len(gpu_t),
                "gpu_seconds_per_key": gpu_t,
                "cpu_ms_per_key": 1e3 * sum(cpu_t) / len(cpu_t), "cpu_cores": THREADS,
                "cpu_kind": "port", "recovered_cpu": ok_cpu,
                "parity": {"bit_exact": restarts == restarts_cpu and ok == ok_cpu,
                           "sample": "every key: recovered flag and restarts used, GPU vs port"},
                "reference_python_seconds_total": 146.0,
                "reference_note": "the Python reference took 146.0 s for this gate (jobs=2) in "
                                  "the build container (SURVEY.md section 6)"})
    plain = G.plain_sct(596)
    logs = cc.LogBigramTable(G.english_logs(), -24.0)
    for k, R in ((10, 5), (15, 10)):
        gpu_t, cpu_t, ok, ok_cpu, agree = [], [], 0, 0, True
        n_cpu = 2 if bounded else 3
        for e in range(3 if quick else 10):
            cipher = cc.sct_encrypt(plain, O.permutation(800 + e, KEYGEN, k))
            cfg = cc.SctSolverConfig(key_length=k, workers=64, climbings=15_000, restarts=R,
                                     global_seed=8000 + e)
            t0 = time.perf_counter()
            best, summ = cc.solve_sct(cipher, logs, cfg,
                                      stop=lambda r: bool(np.array_equal(r.best_text, plain)))
            gpu_t.append(time.perf_counter() - t0)
            ok += bool(np.array_equal(best.best_text, plain))
            if e < n_cpu:  # the CPU port on a sample of the experiments (seconds each)
                t0 = time.perf_counter()
                used = R
                for r in range(R):
                    sc, keys = O.sct_workers([cipher], np.zeros(64, np.int32), [8000 + e] * 64,
                                             [(r << 32) | w for w in range(64)], logs.logs, k,
                                             15_000, threads=THREADS)
                    if r < len(summ):
                        agree &= bool(summ[r].score == float(sc.max()))
                    if np.array_equal(cc.sct_decrypt(cipher, keys[int(np.argmax(sc))]), plain):
                        ok_cpu += 1
                        used = r + 1
                        break
                agree &= used == len(summ)
                cpu_t.append(time.perf_counter() - t0)
        out.append({"config": f"TTR-08-k{k}",
                    "what": f"acceptance #08 SCT: k={k}, 596 letters, 64 x 15k, <= {R} "
                            "restarts, stop on the plaintext",
                    "recovered": ok, "of": len(gpu_t),
                    "gpu_ms_per_key": 1e3 * sum(gpu_t) / len(gpu_t),
                    "gpu_seconds_per_key": gpu_t,
                    "cpu_ms_per_key": 1e3 * sum(cpu_t) / max(1, len(cpu_t)),
                    "cpu_sample_keys": len(cpu_t), "recovered_cpu_sample": ok_cpu,
                    "cpu_cores": THREADS, "cpu_kind": "port",
                    "parity": {"bit_exact": bool(agree),
                               "sample": f"first {len(cpu_t)} keys: every restart's best score "
                                         "and the restarts used, GPU vs port"},
                    "reference_note": "the Python reference took 963.4 s for both #08 gates "
                                      "(20 keys, jobs=2) in the build container (SURVEY.md "
                                      "section 6)"})
    return out


RUNNERS = {"C1": c1, "C1d": c1d, "C3": c3, "C4": c4, "C5": c5, "TTR": ttr}


def run_all(bounded=True, only=None, quick=False):
    """Run the configurations; returns {name: entry-or-list}.  bounded=True keeps the whole
    set near a minute of wall time (fewer restarts on C1/C1d, a 3-point C5 sweep, shorter CPU
    samples) for bench.py's JSON line."""
    out = {}
    for name in (only or list(RUNNERS)):
        t0 = time.perf_counter()
        try:
            r = RUNNERS[name](bounded=bounded, quick=quick)
        except Exception as e:  # noqa: BLE001 - reported in the line, never hides the headline
            r = {"config": name, "error": f"{type(e).__name__}: {e}"}
        for e in (r if isinstance(r, list) else [r]):
            e["wall_s"] = round(time.perf_counter() - t0, 2)
            out.setdefault(e["config"], []).append(e)
    return {k: (v[0] if len(v) == 1 else v) for k, v in out.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--bounded", action="store_true")
    ap.add_argument("--only", default=",".join(RUNNERS))
    args = ap.parse_args()
    engine.set_devices([0])
    for name in args.only.split(","):
        r = RUNNERS[name.strip()](bounded=args.bounded, quick=args.quick)
        for e in (r if isinstance(r, list) else [r]):
            print(json.dumps(e), flush=True)


if __name__ == "__main__":
    main()
