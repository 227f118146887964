"""The reference's end-to-end acceptance gates (reference tests/test_acceptance.py:146-198)
run on the GPU engine, plus key-recovery agreement with the CPU oracle on a sample of the
bench workload (BASELINE.json north_star: "100% key-recovery agreement with the CPU
reference on the test corpus")."""
import numpy as np
import pytest

import paper_2103_13937_b200 as cc
from paper_2103_13937_b200 import engine
from paper_2103_13937_b200.rng import philox_keys
from oracle import oracle as O

pytestmark = pytest.mark.gpu
KEYGEN = 2**32 - 2


def test_07_mas_end_to_end(golden):
    """10 keys, 471 letters, 64 workers x 10k tries, <= 20 restarts, stop on the plaintext,
    >= 8/10 recovered (test_acceptance.py:146-167); every restart's best score equals the
    oracle's."""
    plain = golden.plain_mas(471)
    table = cc.BigramTable(golden.english_scores())
    successes = 0
    for e in range(10):
        key = O.permutation(700 + e, KEYGEN, 26)
        cipher = key[plain]
        cfg = cc.MasSolverConfig(workers=64, climbings=10_000, restarts=20, global_seed=7000 + e)
        best, summ = cc.solve_with_restarts(cipher, table, cfg, jobs=2,
                                            stop=lambda r: bool(np.array_equal(r.best_text, plain)))
        successes += bool(np.array_equal(best.best_text, plain))
        for s in summ:
            want, maps = O.mas_workers([cipher], np.zeros(64, np.int32), [7000 + e] * 64,
                                       [(s.restart << 32) | w for w in range(64)],
                                       table.scores, 10_000)
            assert s.score == int(want.max()), (e, s.restart)
            assert np.array_equal(s.text, maps[int(np.argmax(want))][cipher])
    assert successes >= 8, f"only {successes}/10 recoveries"


@pytest.mark.parametrize("key_length,restarts", [(10, 5), (15, 10)])
def test_08_sct_end_to_end(golden, key_length, restarts):
    """596 letters, 64 workers x 15k tries, >= 7/10 recovered (test_acceptance.py:170-198);
    the first experiment's restarts are checked worker-for-worker against the oracle."""
    plain = golden.plain_sct(596)
    logs = cc.LogBigramTable(golden.english_logs(), -24.0)
    successes = 0
    for e in range(10):
        key = O.permutation(800 + e, KEYGEN, key_length)
        cipher = cc.sct_encrypt(plain, key)
        cfg = cc.SctSolverConfig(key_length=key_length, workers=64, climbings=15_000,
                                 restarts=restarts, global_seed=8000 + e)
        best, summ = cc.solve_sct(cipher, logs, cfg, jobs=2,
                                  stop=lambda r: bool(np.array_equal(r.best_text, plain)))
        successes += bool(np.array_equal(best.best_text, plain))
        if e == 0:
            s = summ[0]
            want, _ = O.sct_workers([cipher], np.zeros(64, np.int32), [8000] * 64,
                                    [(0 << 32) | w for w in range(64)], logs.logs, key_length,
                                    15_000)
            assert s.score == float(want.max())
    assert successes >= 7, f"k={key_length}: only {successes}/10 recoveries"


def test_c2_key_recovery_agrees_with_oracle(golden):
    """A 40-ciphertext sample of the bench workload (C2 recipe: corpus windows of 100-500
    letters, reference key recipe, 64 workers x 10k): the best key of every ciphertext, and
    so its recovered / not-recovered outcome, equals the CPU oracle's."""
    import bench

    plains, ciphers, scores, lengths = bench.make_workload(10_000, 0)
    pick = np.random.default_rng(1).choice(len(ciphers), 40, replace=False)
    cs = [ciphers[i] for i in pick]
    W = 64
    cof = np.repeat(np.arange(len(cs), dtype=np.int32), W)
    seeds = [7000 + int(i) for i in pick for _ in range(W)]
    streams = [w for _ in pick for w in range(W)]
    from paper_2103_13937_b200.rng import philox_key

    keys = np.array([philox_key(s, w) for s, w in zip(seeds, streams)], dtype=np.uint64)
    res = engine.mas_climb(cs, cof, keys, scores, 10_000, group_size=W)
    want_s, want_m = O.mas_workers(cs, cof, seeds, streams, scores, 10_000)
    assert res.scores.tolist() == want_s.tolist()
    agree = 0
    for j, i in enumerate(pick):
        g = int(res.group_best[j])
        assert g == int(np.argmax(want_s[j * W:(j + 1) * W]))
        got_rec = np.array_equal(res.keys[j * W + g].astype(np.int64)[cs[j]], plains[i])
        want_rec = np.array_equal(want_m[j * W + g][cs[j]], plains[i])
        agree += got_rec == want_rec
    assert agree == len(pick)
