#!/usr/bin/env python
"""Throughput and quality on BASELINE.json's other configurations (bench.py measures the
headline, configs[1] = C2).  One JSON line per measurement on stdout.

  C1  MAS, one 300-letter held-out ciphertext (acceptance #07 recipe, key_seed 700), bigram,
      64 workers x 10,000 climbings x R restarts; time-to-recover through solve_with_restarts
      with stop-on-plaintext and the exact early exit.
  C1d the deterministic best-neighbour solver on the same ciphertext (mas.py:140-169),
      R restarts x 500 iterations x 325 candidates.
  C3  SCT, key lengths 5..20, 1,000 ciphertexts of 400 letters, trigram log table.
  C4  MAS, 60-100 letter ciphertexts, quadgram (uint16 quantised log table, read via L2),
      one worker per restart.
  C5  evals/s vs workers (1e3..1e6) and n-gram order 2/3/4.

Every timed call goes through the public engine API from host buffers (H2D + D2H inside the
timed region) after a warm-up call; evals count executed fitness evaluations only.  The CPU
column is the C oracle (oracle/cc_oracle.c, a port of the reference algorithm) on all host
cores over a bounded sample of the same work.

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
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import golden_data as G  # noqa: E402
import paper_2103_13937_b200 as cc  # noqa: E402
from paper_2103_13937_b200 import engine  # noqa: E402
from paper_2103_13937_b200.rng import philox_keys  # noqa: E402

KEYGEN = 2**32 - 2
THREADS = os.cpu_count() or 1


def emit(d):
    print(json.dumps(d), flush=True)


def timed(fn, reps=1):
    fn()  # warm-up (also loads tables / allocates scratch)
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    return out, (time.perf_counter() - t0) / reps


def corpus_text():
    return "".join(chr(97 + int(x)) for x in G.corpus())


def cpu_rate(fn, evals_of, budget_s=4.0):
    """Run fn(m) for growing m until it takes >= budget_s; return evals/s."""
    m = 1
    while True:
        t0 = time.perf_counter()
        fn(m)
        dt = time.perf_counter() - t0
        if dt >= budget_s or m >= 1 << 20:
            return evals_of(m) / dt, m
        m = max(m + 1, int(m * min(8.0, 1.5 * budget_s / max(dt, 1e-3))))


def c1(args):
    from oracle import oracle as O

    plain = G.plain_mas(300)
    key = O.permutation(700, KEYGEN, 26)
    cipher = key[plain]
    table = cc.BigramTable(G.english_scores())
    R = 2000 if args.quick else 10_000
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
                           lambda m: m * THREADS * K)
    true_score = int(cc.score_text(plain, table))
    emit({"config": "C1", "what": "MAS n=300 bigram, 64 workers x 10k climbings x restarts",
          "restarts": R, "evals": evals, "seconds": dt, "evals_per_s": evals / dt,
          "cpu_evals_per_s": rate_cpu, "cpu_cores": THREADS,
          "best_score": int(res.scores[best]), "true_plaintext_score": true_score,
          "restarts_recovering_plaintext": int(sum(
              np.array_equal(res.keys[r * W + int(res.group_best[r])].astype(np.int64)[cipher], plain)
              for r in range(R)))})
    # time-to-recover key through the public API: restarts until the plaintext comes out
    cfg = cc.MasSolverConfig(workers=W, climbings=K, restarts=R, global_seed=7000)
    t0 = time.perf_counter()
    best_res, summ = cc.solve_with_restarts(cipher, table, cfg,
                                            stop=lambda r: np.array_equal(r.best_text, plain))
    ttr = time.perf_counter() - t0
    emit({"config": "C1", "what": "time-to-recover-key (solve_with_restarts, stop on plaintext, "
                                  "exact early exit)",
          "recovered": bool(np.array_equal(summ[-1].text, plain)), "restarts_used": len(summ),
          "seconds": ttr})


def c1d(args):
    from oracle import oracle as O

    plain = G.plain_mas(300)
    cipher = O.permutation(700, KEYGEN, 26)[plain]
    table = cc.BigramTable(G.english_scores())
    R = 2000 if args.quick else 20_000
    keys = philox_keys([606], [(r << 32) | (2**32 - 1) for r in range(R)])
    res, dt = timed(lambda: engine.mas_det_solve([cipher], np.zeros(R, np.int32), keys, table.scores,
                                                 500))
    evals = R * 500 * 325
    rate_cpu, m = cpu_rate(lambda m: [O.solve_deterministic(cipher, table.scores, 500, 606, r)
                                      for r in range(m)], lambda m: m * 500 * 325, budget_s=3.0)
    emit({"config": "C1d", "what": "deterministic best-neighbour MAS n=300, 500 iterations x 325 "
                                   "candidates per restart", "restarts": R,
          "candidate_evals": evals, "seconds": dt, "evals_per_s": evals / dt,
          "cpu_evals_per_s_1core": rate_cpu,
          "best_score": int(res.scores.max()),
          "recovered": bool(np.array_equal(res.maps[int(np.argmax(res.scores))].astype(np.int64)[cipher],
                                           plain))})


def c3(args):
    from oracle import oracle as O

    l3 = cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus_text(), 3))
    corpus = G.corpus()
    n_c = 1000
    W, K = (8, 1000) if args.quick else (32, 15_000)  # climbings 15,000
    ks = list(range(5, 21))
    ciphers, plains, kofc = [], [], []
    for i in range(n_c):
        k = 5 + i % len(ks)
        off = int(np.random.default_rng(300000 + i).integers(0, corpus.size - 400))
        p = corpus[off:off + 400]
        key = O.permutation(300000 + i, KEYGEN, k)
        plains.append(p)
        ciphers.append(cc.sct_encrypt(p, key))
        kofc.append(k)
    # one launch for the whole ragged batch (per-worker key length)
    cof = np.repeat(np.arange(n_c, dtype=np.int32), W)
    klens = np.repeat(np.array(kofc, dtype=np.int32), W)
    keys = philox_keys([9000], list(range(cof.size)))
    res, total_s = timed(lambda: engine.sct_climb(ciphers, cof, keys, l3.logs, klens, K, order=3,
                                                  group_size=W))
    total_evals = cof.size * K
    rec, rows = 0, []
    for k in ks:
        idx = [j for j in range(n_c) if kofc[j] == k]
        ok = sum(np.array_equal(cc.sct_decrypt(ciphers[j], res.keys[j * W + int(res.group_best[j]), :k]
                                               .astype(np.int64)), plains[j]) for j in idx)
        rec += ok
        rows.append({"k": k, "ciphers": len(idx), "recovered": int(ok)})
    c0 = ciphers[0]
    rate_cpu, m = cpu_rate(lambda m: O.sct_workers([c0], np.zeros(m * THREADS, np.int32),
                                                   [9000] * (m * THREADS), list(range(m * THREADS)),
                                                   l3.logs, 20, 200, order=3, threads=THREADS),
                           lambda m: m * THREADS * 200)
    emit({"config": "C3", "what": "SCT k=5..20, 1000 ciphertexts x 400 letters, trigram log table",
          "workers_per_cipher": W, "climbings": K, "launches": "one (ragged key lengths)",
          "evals": total_evals, "seconds": total_s,
          "evals_per_s": total_evals / total_s, "recovered": rec, "of": n_c,
          "cpu_evals_per_s": rate_cpu, "cpu_cores": THREADS, "per_k": rows})


def c4(args):
    from oracle import oracle as O

    q4 = cc.quantize_log_table(cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus_text(), 4)))
    n_c = 125
    R = 200 if args.quick else 1000
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
    res, dt = timed(lambda: engine.mas_climb(ciphers, cof, keys, q4.scores, K, order=4, group_size=R,
                                             computed=True))
    evals = cof.size * K
    ok = sum(np.array_equal(res.keys[j * R + int(res.group_best[j])].astype(np.int64)[ciphers[j]],
                            plains[j]) for j in range(n_c))
    rate_cpu, m = cpu_rate(lambda m: O.ngram_workers([ciphers[0]], np.zeros(m * THREADS, np.int32),
                                                     [4000] * (m * THREADS), list(range(m * THREADS)),
                                                     4, q4.scores, 2000, threads=THREADS),
                           lambda m: m * THREADS * 2000)
    emit({"config": "C4", "what": "MAS 60-100 letters, quadgram uint16 table via L2, one worker per "
                                  "restart", "ciphers": n_c, "restarts_per_cipher": R,
          "climbings": K, "evals": evals, "seconds": dt, "evals_per_s": evals / dt,
          "computed_by_walk": float(res.computed.sum() / evals),
          "recovered": int(ok), "of": n_c, "cpu_evals_per_s": rate_cpu, "cpu_cores": THREADS,
          "cpu_kind": "oracle port, full rescore per try"})


def c5(args):
    corpus = corpus_text()
    tabs = {2: cc.BigramTable(G.english_scores()).scores}
    for o in (3, 4):
        tabs[o] = cc.quantize_log_table(cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus, o))).scores
    plain = G.plain_mas(300)
    cipher = np.random.default_rng(1).permutation(26)[plain]
    K = 10_000
    sizes = [1000, 10_000, 100_000] + ([] if args.quick else [1_000_000, 10_000_000])
    key_cache = {}
    for order in (2, 3, 4):
        for n in sizes:
            if n not in key_cache:
                key_cache[n] = philox_keys([5], list(range(n)))
            keys = key_cache[n]
            res, dt = timed(lambda: engine.mas_climb([cipher], np.zeros(n, np.int32), keys,
                                                     tabs[order], K, order=order,
                                                     computed=order > 2))
            line = {"config": "C5", "order": order, "workers": n, "climbings": K, "text_len": 300,
                    "evals_per_s": n * K / dt, "seconds": dt}
            if order > 2:
                line["computed_by_walk"] = float(res.computed.sum() / (n * K))
            emit(line)


def ttr(args):
    """Time to recover the key on the reference's acceptance recipes (tests/test_acceptance.py
    :146-198; BASELINE.json metric "time-to-recover key"): MAS #07 (471 letters, 10 keys,
    64 workers x 10k, <= 20 restarts) and SCT #08 (596 letters, k = 10 / 15, 64 x 15k,
    <= 5 / 10 restarts), stop on the exact plaintext, through the public API.  CPU column:
    the C oracle port on all host cores running the same restarts until the same stop."""
    from oracle import oracle as O

    plain = G.plain_mas(471)
    table = cc.BigramTable(G.english_scores())
    # warm-up (context, module load) outside the timed solves
    cc.solve_with_restarts(O.permutation(1, KEYGEN, 26)[plain], table,
                           cc.MasSolverConfig(workers=64, climbings=1000, restarts=2))
    gpu_t, cpu_t, ok, ok_cpu, restarts = [], [], 0, 0, []
    for e in range(10 if not args.quick else 3):
        cipher = O.permutation(700 + e, KEYGEN, 26)[plain]
        cfg = cc.MasSolverConfig(workers=64, climbings=10_000, restarts=20, global_seed=7000 + e)
        t0 = time.perf_counter()
        best, summ = cc.solve_with_restarts(cipher, table, cfg,
                                            stop=lambda r: bool(np.array_equal(r.best_text, plain)))
        gpu_t.append(time.perf_counter() - t0)
        ok += bool(np.array_equal(best.best_text, plain))
        restarts.append(len(summ))
        t0 = time.perf_counter()
        for r in range(20):
            s, m = O.mas_workers([cipher], np.zeros(64, np.int32), [7000 + e] * 64,
                                 [(r << 32) | w for w in range(64)], table.scores, 10_000,
                                 threads=THREADS)
            if np.array_equal(m[int(np.argmax(s))][cipher], plain):
                ok_cpu += 1
                break
        cpu_t.append(time.perf_counter() - t0)
    emit({"config": "TTR", "what": "acceptance #07 MAS: 10 keys, 471 letters, 64 x 10k, <= 20 "
                                   "restarts, stop on the plaintext",
          "recovered": ok, "recovered_cpu": ok_cpu, "of": len(gpu_t),
          "restarts_used": restarts, "gpu_seconds_total": sum(gpu_t),
          "gpu_seconds_per_key": gpu_t, "cpu_seconds_total": sum(cpu_t), "cpu_cores": THREADS,
          "reference_python_seconds_total": 146.0,
          "reference_note": "the Python reference took 146.0 s for this gate (jobs=2) in the "
                            "build container (SURVEY.md section 6)"})
    plain = G.plain_sct(596)
    logs = cc.LogBigramTable(G.english_logs(), -24.0)
    for k, R in ((10, 5), (15, 10)):
        gpu_t, cpu_t, ok, ok_cpu = [], [], 0, 0
        for e in range(10 if not args.quick else 3):
            cipher = cc.sct_encrypt(plain, O.permutation(800 + e, KEYGEN, k))
            cfg = cc.SctSolverConfig(key_length=k, workers=64, climbings=15_000, restarts=R,
                                     global_seed=8000 + e)
            t0 = time.perf_counter()
            best, _ = cc.solve_sct(cipher, logs, cfg,
                                   stop=lambda r: bool(np.array_equal(r.best_text, plain)))
            gpu_t.append(time.perf_counter() - t0)
            ok += bool(np.array_equal(best.best_text, plain))
            if e < 3:  # the CPU port on a sample of the experiments (it takes seconds each)
                t0 = time.perf_counter()
                for r in range(R):
                    sc, keys = O.sct_workers([cipher], np.zeros(64, np.int32), [8000 + e] * 64,
                                             [(r << 32) | w for w in range(64)], logs.logs, k,
                                             15_000, threads=THREADS)
                    if np.array_equal(cc.sct_decrypt(cipher, keys[int(np.argmax(sc))]), plain):
                        ok_cpu += 1
                        break
                cpu_t.append(time.perf_counter() - t0)
        emit({"config": "TTR", "what": f"acceptance #08 SCT: k={k}, 596 letters, 64 x 15k, "
                                       f"<= {R} restarts, stop on the plaintext",
              "recovered": ok, "of": len(gpu_t), "gpu_seconds_total": sum(gpu_t),
              "gpu_seconds_per_key": gpu_t, "cpu_seconds_per_key_sample": cpu_t,
              "cpu_recovered_sample": ok_cpu, "cpu_cores": THREADS,
              "reference_note": "the Python reference took 963.4 s for both #08 gates (20 keys, "
                                "jobs=2) in the build container (SURVEY.md section 6)"})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="C1,C1d,C3,C4,C5,TTR")
    args = ap.parse_args()
    engine.set_devices([0])
    for name in args.only.split(","):
        {"C1": c1, "C1d": c1d, "C3": c3, "C4": c4, "C5": c5, "TTR": ttr}[name.strip()](args)


if __name__ == "__main__":
    main()
