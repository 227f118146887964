"""GPU parity: the CUDA engine (through the C ABI) vs the reference's golden outputs and
the pinned CPU oracle.  Integer and index work must be bit-exact; SCT float64 scores
must be bit-exact too (numpy pairwise order), so no tolerance appears below."""
import numpy as np
import pytest

import paper_2103_13937_b200 as cc
from paper_2103_13937_b200 import engine
from paper_2103_13937_b200.rng import philox_key, philox_keys
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    from paper_2103_13937_b200 import _lib

    if _lib.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


# ------------------------------------------------------------------ rng (rng.py:58-97)
def test_philox_uniforms_match_reference(golden):
    g = golden.load("rng")
    for i, (s, w) in enumerate(zip(g["keys_seed"], g["keys_stream"])):
        got = cc.rng.draws(int(s), int(w), 300)
        assert np.array_equal(got, g["uniforms"][i]), (s, w)
        for skip in (1, 3, 5, 130):
            assert np.array_equal(cc.rng.draws(int(s), int(w), 40, skip=skip),
                                  g["uniforms"][i][skip:skip + 40])


def test_int_below_exact_against_float64():
    from paper_2103_13937_b200 import _lib

    ctx = _lib.context(0)
    n = 1 << 20
    for seed, stream in [(5, 9), (2**63 - 1, (7 << 32) | 3)]:
        k0, k1 = philox_key(seed, stream)
        u = np.empty(n)
        _lib.check(_lib.load().ccg_philox_uniform(ctx.handle, k0, k1, 0, n, _lib.ptr(u)), "u")
        for bound in (1, 2, 3, 7, 26, 99, 100, 1999, 2**20 + 3, 2**31 - 1):
            got = np.empty(n, dtype=np.int64)
            _lib.check(_lib.load().ccg_philox_int_below(ctx.handle, k0, k1, 0, bound, n,
                                                        _lib.ptr(got)), "ib")
            assert np.array_equal(got, (u * bound).astype(np.int64)), bound


def test_worker_rng_api(golden):
    g = golden.load("rng")
    for b in (2, 3, 10, 26):
        st = cc.WorkerRng(17, b)
        got = np.array([st.next_distinct_pair(b) for _ in range(2000)])
        assert np.array_equal(got, g[f"pairs_{b}"])
    for n in (1, 2, 3, 5, 10, 26, 40, 64):
        assert np.array_equal(cc.WorkerRng(19, n).permutation(n), g[f"perm_{n}"])


# ------------------------------------------------------------------ fitness
def test_score_text_batch_matches_reference(golden):
    g = golden.load("scoring")
    texts = golden.scoring_texts()
    rnd = cc.BigramTable(g["rnd_table"])
    eng = cc.BigramTable(golden.english_scores())
    assert np.array_equal(cc.score_text_batch(texts, rnd), g["int_scores"])
    assert np.array_equal(cc.score_text_batch(texts, eng), g["eng_scores"])


def test_log_score_text_bit_exact(golden):
    g = golden.load("scoring")
    logs = cc.LogBigramTable(golden.english_logs(), -24.0)
    got = cc.log_score_text_batch(golden.scoring_texts(), logs)
    assert got.tolist() == g["log_scores"].tolist()  # bit-exact float64
    assert cc.log_score_text(np.array([3]), logs) == 0.0


def test_log_score_random_lengths_vs_oracle():
    rng = np.random.default_rng(7)
    logs = -rng.random(676) * 20 - 1
    tab = cc.LogBigramTable(logs, -30.0)
    lens = list(range(0, 300)) + [511, 512, 513, 1000, 1025, 1500, 2047, 2048, 2049, 3000, 4096]
    texts = [rng.integers(0, 26, L) for L in lens]
    got = cc.log_score_text_batch(texts, tab)
    want = [O.log_score_text(t, logs) for t in texts]
    assert got.tolist() == want


def test_delta_acceptance_05(golden):
    table, cases, want = golden.delta_cases()
    got = engine.mas_delta_batch([c[0] for c in cases], [(c[1], c[2]) for c in cases], table)
    assert np.array_equal(got, want)


def test_delta_wide_tables_vs_oracle():
    rng = np.random.default_rng(8)
    for high in (70_000, 2**40):
        table = rng.integers(0, high, 676)
        texts = [rng.integers(0, 26, int(rng.integers(2, 400))) for _ in range(300)]
        pairs = [tuple(rng.choice(26, 2, replace=False)) for _ in texts]
        got = engine.mas_delta_batch(texts, pairs, table)
        want = [O.text_swap_delta(t, a, b, table) for t, (a, b) in zip(texts, pairs)]
        assert got.tolist() == want


def test_swap_delta_on_count_matrices():
    rng = np.random.default_rng(9)
    for signed in (False, True):
        S = rng.integers(-500 if signed else 0, 900, 676)
        for _ in range(50):
            t = rng.integers(0, 26, int(rng.integers(2, 300)))
            a, b = (int(v) for v in rng.choice(26, 2, replace=False))
            counts = cc.bigram_count_matrix(t)
            assert cc.swap_delta(counts, a, b, S.reshape(26, 26)) == O.text_swap_delta(t, a, b, S)


# ------------------------------------------------------------------ MAS climb
def test_stochastic_worker_golden(golden):
    for cipher, table, climb, seed, stream, want_text, want_score in golden.mas_worker_cases(
            O.permutation):
        st = cc.WorkerRng(seed, stream)
        text, score = cc.stochastic_worker(cipher, cc.BigramTable(table), climb, st)
        assert score == want_score
        assert np.array_equal(text, want_text)


def test_stochastic_worker_advances_state_like_reference():
    # after a worker, the state continues exactly where the reference's generator would
    t = np.random.default_rng(1).integers(0, 26, 120)
    tab = cc.BigramTable(np.random.default_rng(2).integers(0, 500, 676))
    st = cc.WorkerRng(3, 4)
    cc.stochastic_worker(t, tab, 700, st)
    # the oracle consumes the same number of draws: replay by counting pairs
    pairs = O.distinct_pairs(3, 4, 26, 700)
    u = O.uniforms(3, 4, 2000)
    ints = (u * 26).astype(int)
    pos = 0
    for _ in range(700):
        a = ints[pos]; pos += 1
        b = ints[pos]; pos += 1
        while b == a:
            b = ints[pos]; pos += 1
    assert st.position == pos
    assert pairs.shape == (700, 2)
    # and a second worker from the advanced state matches the oracle with skip
    text2, score2 = cc.stochastic_worker(t, tab, 300, st)
    o_text, o_score, _, _ = O.stochastic_worker(t, tab.scores, 300, 3, 4, skip=pos)
    assert score2 == o_score and np.array_equal(text2, o_text)


@pytest.mark.parametrize("early_exit", [False, True])
def test_mas_solve_golden_per_worker(golden, early_exit):
    g = golden.load("mas_solve")
    cipher = g["cipher"].astype(np.int64)
    eng = golden.english_scores()
    for r in range(2):
        keys = philox_keys([7000], [(r << 32) | w for w in range(64)])
        res = engine.mas_climb([cipher], np.zeros(64, np.int32), keys, eng, 10_000, group_size=64,
                               early_exit=early_exit, tries_done=True)
        assert res.scores.tolist() == g["per_worker"][r].tolist()
        best = int(res.group_best[0])
        assert best == int(np.argmax(g["per_worker"][r]))
        assert np.array_equal(res.keys[best][cipher], g["best_text"][r])
        if early_exit:
            assert res.tries_done.max() <= 10_000
        else:
            assert (res.tries_done == 10_000).all()


def test_solve_stochastic_api_golden(golden):
    g = golden.load("mas_solve")
    cipher = g["cipher"].astype(np.int64)
    table = cc.BigramTable(golden.english_scores())
    cfg = cc.MasSolverConfig(workers=64, climbings=10_000, restarts=20, global_seed=7000)
    for r in range(2):
        res = cc.solve_stochastic(cipher, table, cfg, restart=r)
        assert res.per_worker_scores == g["per_worker"][r].tolist()
        assert res.best_score == g["best_score"][r]
        assert np.array_equal(res.best_text, g["best_text"][r])


def test_mas_random_batch_vs_oracle():
    rng = np.random.default_rng(11)
    ciphers = [rng.integers(0, 26, int(L)) for L in rng.integers(2, 700, 40)]
    ciphers[0] = np.array([4, 4, 9])  # tiny
    tables = [rng.integers(0, 900, 676), rng.integers(0, 65_536, 676), rng.integers(0, 10**9, 676)]
    for table in tables:
        n = 160
        cof = rng.integers(0, len(ciphers), n).astype(np.int32)
        seeds = rng.integers(0, 2**62, n)
        streams = rng.integers(0, 2**40, n)
        keys = philox_keys(seeds.tolist(), streams.tolist())
        for early in (False, True):
            res = engine.mas_climb(ciphers, cof, keys, table, 1500, early_exit=early)
            want_s, want_m = O.mas_workers(ciphers, cof, seeds.tolist(), streams.tolist(), table,
                                           1500)
            assert res.scores.tolist() == want_s.tolist()
            assert np.array_equal(res.keys.astype(np.int64), want_m)


@pytest.mark.parametrize("tmax", [900, 32_767, 32_768])
def test_mas_budget_edges_and_bookkeeping(tmax):
    """Odd and tiny budgets, stream skips, and the T-form gate (max S <= 32767) on both
    sides: scores, maps, draw positions and last accepts equal the oracle's."""
    rng = np.random.default_rng(tmax)
    ciphers = [rng.integers(0, 26, int(L)) for L in (2, 3, 17, 160, 499)]
    table = rng.integers(0, tmax + 1, 676)
    table[int(rng.integers(676))] = tmax
    for climb in (0, 1, 2, 3, 7, 255, 257, 1001):
        for skip in (0, 5):
            n = len(ciphers)
            seeds, streams = [42] * n, [(3 << 32) | w for w in range(n)]
            keys = philox_keys(seeds, streams)
            res = engine.mas_climb(ciphers, np.arange(n, dtype=np.int32), keys, table, climb,
                                   skips=np.full(n, skip, np.uint64), draws_used=True,
                                   last_accept=True)
            for w, c in enumerate(ciphers):
                o_text, o_score, o_map, o_last = O.stochastic_worker(c, table, climb, seeds[w],
                                                                     streams[w], skip=skip)
                assert res.scores[w] == o_score, (climb, skip, w)
                assert np.array_equal(res.keys[w].astype(np.int64)[c], o_text)
                assert res.last_accept[w] == o_last
                pairs_pos = skip
                if climb:
                    ints = (O.uniforms(seeds[w], streams[w], skip + 4 * climb + 64)[skip:] * 26)
                    ints = ints.astype(int)
                    pos = 0
                    for _ in range(climb):
                        a = ints[pos]; pos += 1
                        b = ints[pos]; pos += 1
                        while b == a:
                            b = ints[pos]; pos += 1
                    pairs_pos = skip + pos
                assert int(res.draws_used[w]) == pairs_pos


def test_mas_results_independent_of_device_split():
    rng = np.random.default_rng(12)
    ciphers = [rng.integers(0, 26, 300) for _ in range(3)]
    table = rng.integers(0, 900, 676)
    n = 96
    keys = philox_keys([5], list(range(n)))
    cof = np.repeat(np.arange(3), 32).astype(np.int32)
    one = engine.mas_climb(ciphers, cof, keys, table, 2000, group_size=32)
    two = engine.mas_climb(ciphers, cof, keys, table, 2000, group_size=32, devices_=[0, 0, 0])
    assert np.array_equal(one.scores, two.scores)
    assert np.array_equal(one.keys, two.keys)
    assert np.array_equal(one.group_best, two.group_best)


@pytest.mark.parametrize("order,kmax,m", [(2, 40, 40), (3, 40, 40), (2, 32, 40), (3, 17, 40),
                                           (2, 40, 100), (3, 17, 100)])
def test_sct_speculative_kernel_matches_warp_kernel(order, kmax, m):
    """Few workers run on the speculative latency kernels (ccg_sct.cu: up to 74 workers on the
    two-SM sct_climb_pair_kernel, up to one per SM on sct_climb_chain_kernel, and
    sct_climb_spec_kernel with speculate="replay"): every output equals the
    one-warp-per-worker kernel's, for ragged key lengths and budgets that are not multiples
    of the speculation depth."""
    rng = np.random.default_rng(90 + order)
    n_len = 333
    cs = [rng.integers(0, 26, n_len) for _ in range(3)]
    logs = -rng.random(26**order) * 20 - 1
    cof = rng.integers(0, 3, m).astype(np.int32)
    klens = rng.integers(2, kmax + 1, m).astype(np.int32)
    klens[0] = kmax  # the batch maximum picks the warp kernel's narrow (<= 32) or wide variant
    keys = philox_keys([23], list(range(m)))
    for climb in (0, 1, 2, 3, 5, 417):
        kw = dict(order=order, draws_used=True, last_accept=True, tries_done=True)
        a = engine.sct_climb(cs, cof, keys, logs, klens, climb, **kw)
        r = engine.sct_climb(cs, cof, keys, logs, klens, climb, speculate="replay", **kw)
        b = engine.sct_climb(cs, cof, keys, logs, klens, climb, speculate=False, **kw)
        for x in (a, r):
            assert x.scores.tolist() == b.scores.tolist(), climb
            for i in range(m):
                assert np.array_equal(x.keys[i, :klens[i]], b.keys[i, :klens[i]]), (climb, i)
            assert np.array_equal(x.draws_used, b.draws_used), climb
            assert np.array_equal(x.last_accept, b.last_accept), climb
            assert np.array_equal(x.tries_done, b.tries_done), climb


@pytest.mark.parametrize("k,hops", [(2, (1, 1)), (3, (3, 1)), (7, (2, 3)), (12, (3, 3)), (64, (3, 2))])
def test_sct_chain_kernel_long_climbs(k, hops):
    """The chain-parsed latency kernel across many parse chunks (4,096 draws each) and odd
    operator mixes: identical to the one-warp kernel for every output."""
    rng = np.random.default_rng(500 + k)
    n_len = 200 if k < 64 else 300
    cs = [rng.integers(0, 26, n_len) for _ in range(2)]
    logs = -rng.random(676) * 20 - 1
    m = 6
    cof = (np.arange(m) % 2).astype(np.int32)
    keys = philox_keys([77], list(range(m)))
    kw = dict(draws_used=True, last_accept=True, tries_done=True, op1_hop=hops[0],
              op2_hop=hops[1], p1=20, p2=55)
    a = engine.sct_climb(cs, cof, keys, logs, k, 5000, **kw)
    b = engine.sct_climb(cs, cof, keys, logs, k, 5000, speculate=False, **kw)
    assert a.scores.tolist() == b.scores.tolist()
    assert np.array_equal(a.keys, b.keys)
    assert np.array_equal(a.draws_used, b.draws_used)
    assert np.array_equal(a.last_accept, b.last_accept)
    assert np.array_equal(a.tries_done, b.tries_done)


def test_restarts_stop_and_prefix(golden):
    table = cc.BigramTable(np.random.default_rng(29).integers(0, 500, 676))
    cipher = np.random.default_rng(30).integers(0, 26, 120)
    short = cc.MasSolverConfig(workers=4, climbings=800, restarts=2, global_seed=3)
    longer = cc.MasSolverConfig(workers=4, climbings=800, restarts=4, global_seed=3)
    b1, r1 = cc.solve_with_restarts(cipher, table, short)
    b2, r2 = cc.solve_with_restarts(cipher, table, longer)
    assert [r.score for r in r2[:2]] == [r.score for r in r1]
    assert b2.best_score >= b1.best_score
    assert [r.restart for r in r2] == [0, 1, 2, 3]
    _, runs = cc.solve_with_restarts(cipher, table, longer, stop=lambda r: True)
    assert len(runs) == 1
    # each restart equals the oracle's workers on streams (r << 32) | w
    for r in range(4):
        want, _ = O.mas_workers([cipher], np.zeros(4, np.int32), [3] * 4,
                                [(r << 32) | w for w in range(4)], table.scores, 800)
        assert r2[r].score == want.max()


# ------------------------------------------------------------------ SCT
def test_sct_score_batch_vs_oracle():
    rng = np.random.default_rng(13)
    logs = -rng.random(676) * 20 - 1
    cases = []
    for k in list(range(1, 41)) + [47, 63, 64]:
        for n in (k, k + 1, 2 * k + 3, 7 * k + 5, 400, 596, 1024, 2049):
            if n >= k:
                cases.append((k, n))
    for k, n in cases:
        cipher = rng.integers(0, 26, n)
        keys = np.array([rng.permutation(k) for _ in range(3)], dtype=np.uint8)
        got = engine.sct_score_batch([cipher], np.zeros(3, np.int32), keys, logs)
        want = [O.sct_score(cipher, logs, kk) for kk in keys]
        assert got.tolist() == want, (k, n)


def test_sct_worker_golden(golden):
    for cipher, logs, k, climb, seed, stream, want_key, want_score in golden.sct_worker_cases():
        cfg = cc.SctSolverConfig(key_length=k, climbings=climb, workers=1)
        lt = cc.LogBigramTable(logs, float(np.min(logs)))
        key, score = cc.sct_worker(cipher, lt, cfg, cc.WorkerRng(seed, stream))
        assert np.array_equal(key, want_key), (k, cipher.size)
        assert score == want_score


def test_sct_solve_golden(golden):
    g = golden.load("sct_solve")
    cipher = g["cipher"].astype(np.int64)
    logs = cc.LogBigramTable(golden.english_logs(), -24.0)
    cfg = cc.SctSolverConfig(key_length=10, workers=64, climbings=15_000, restarts=1,
                             global_seed=8000)
    best, runs = cc.solve_sct(cipher, logs, cfg)
    assert best.per_worker_scores == g["per_worker"].tolist()
    assert np.array_equal(best.best_key, g["best_key"])
    assert np.array_equal(best.best_text, g["best_text"])
    assert best.best_score == float(g["best_score"])
    assert len(runs) == 1


def test_sct_random_workers_vs_oracle():
    rng = np.random.default_rng(14)
    logs = -rng.random(676) * 20 - 1
    for k, n in [(2, 9), (3, 40), (5, 400), (8, 8), (12, 100), (20, 400), (31, 300), (33, 500),
                 (40, 800), (64, 700), (7, 1500)]:
        ciphers = [rng.integers(0, 26, n) for _ in range(2)]
        m = 24
        cof = (np.arange(m) % 2).astype(np.int32)
        seeds = rng.integers(0, 2**62, m)
        streams = rng.integers(0, 2**40, m)
        p1, p2 = sorted(rng.integers(0, 101, 2).tolist())
        h1, h2 = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        res = engine.sct_climb(ciphers, cof, philox_keys(seeds.tolist(), streams.tolist()), logs, k,
                               400, p1=p1, p2=p2, op1_hop=h1, op2_hop=h2)
        want_s, want_k = O.sct_workers(ciphers, cof, seeds.tolist(), streams.tolist(), logs, k, 400,
                                       p1=p1, p2=p2, op1_hop=h1, op2_hop=h2)
        assert res.scores.tolist() == want_s.tolist(), (k, n)
        assert np.array_equal(res.keys.astype(np.int64), want_k), (k, n)


def test_sct_end_to_end_small(golden):
    plain = golden.plain_sct()[:80]
    key = np.random.default_rng(52).permutation(4)
    cipher = cc.sct_encrypt(plain, key)
    logs = cc.LogBigramTable(golden.english_logs(), -24.0)
    cfg = cc.SctSolverConfig(key_length=4, workers=8, climbings=2000, global_seed=12)
    best, _ = cc.solve_sct(cipher, logs, cfg)
    assert best.best_score >= O.log_score_text(plain, golden.english_logs())
    assert np.array_equal(best.best_text, plain)


# ------------------------------------------------------------------ acceptance-style end to end
def test_mas_acceptance_07_shape(golden):
    """tests/test_acceptance.py:146-167 (first 3 experiments): GPU run must reproduce the
    oracle's restart-by-restart outcome and recover the plaintext."""
    plain = golden.plain_mas(471)
    table = cc.BigramTable(golden.english_scores())
    ok = 0
    for e in range(3):
        key = O.permutation(700 + e, cc.KEYGEN_STREAM, 26)
        cipher = key[plain]
        cfg = cc.MasSolverConfig(workers=64, climbings=10_000, restarts=20, global_seed=7000 + e)
        best, runs = cc.solve_with_restarts(cipher, table, cfg,
                                            stop=lambda r: bool(np.array_equal(r.best_text, plain)))
        ok += bool(np.array_equal(best.best_text, plain))
        last = runs[-1].restart
        want, _ = O.mas_workers([cipher], np.zeros(64, np.int32), [7000 + e] * 64,
                                [(last << 32) | w for w in range(64)], table.scores, 10_000)
        assert runs[-1].score == want.max()
    assert ok >= 2


# ------------------------------------------------------------------ deterministic MAS (mas.py:84-169)
def test_det_step_matches_reference(golden):
    cases = golden.det_step_cases()
    for text, pivot, table, score, index, cand in cases:
        got_t, got_s, got_i = cc.deterministic_step(text, pivot, cc.BigramTable(table))
        assert (got_s, got_i) == (score, index)
        assert np.array_equal(got_t, cand)


def test_det_step_all_scores_vs_oracle():
    # every one of the 325 pair-worker scores, including excluded ones and wide tables
    rng = np.random.default_rng(31)
    texts, pivots, tables = [], [], []
    for i in range(60):
        L = int(rng.integers(2, 700))
        t = rng.integers(0, 26, L)
        if np.unique(t).size < 2:
            t[0], t[-1] = 3, 4
        texts.append(t)
        pivots.append(tuple(int(v) for v in rng.choice(np.unique(t), 2, replace=False)))
    for hi in (900, 40_000, 2**40):
        table = rng.integers(0, hi, 676)
        got = engine.mas_det_step_batch(texts, pivots, table)
        for t, pv, row in zip(texts, pivots, got):
            want, _, _ = O.det_step(t, pv, table)
            assert np.array_equal(row, want)


def test_det_step_validation():
    table = cc.BigramTable(np.arange(676))
    with pytest.raises(ValueError):
        cc.deterministic_step(cc.map_text("abcabc"), (0, 0), table)
    with pytest.raises(ValueError):
        cc.deterministic_step(cc.map_text("abcabc"), (0, 25), table)


def test_solve_deterministic_matches_reference(golden):
    for cipher, table, seed, r, iters, text, score, hist in golden.det_run_cases():
        cfg = cc.MasSolverConfig(mode="deterministic", workers=325, iterations=iters,
                                 global_seed=seed)
        res = cc.solve_deterministic(cipher, cc.BigramTable(table), cfg, restart=r)
        assert res.best_score == score and res.history == hist
        assert np.array_equal(res.best_text, text)
        assert res.per_worker_scores == []


def test_solve_deterministic_batch_vs_oracle():
    # many jobs in one launch, random tables (narrow and wide accumulators), vs the oracle
    rng = np.random.default_rng(44)
    for hi in (700, 3_000_000):
        table = rng.integers(0, hi, 676)
        ciphers = [rng.integers(0, 26, int(rng.integers(2, 400))) for _ in range(24)]
        for c in ciphers:
            if np.unique(c).size < 2:
                c[0], c[-1] = 1, 2
        seed = int(rng.integers(0, 2**63))
        cof = np.repeat(np.arange(len(ciphers), dtype=np.int32), 2)
        restarts = [0, 3] * len(ciphers)
        keys = philox_keys([seed], [((r << 32) | (2**32 - 1)) for r in restarts])
        res = engine.mas_det_solve(ciphers, cof, keys, table, 120)
        for j, (c, r) in enumerate(zip(cof, restarts)):
            t, s, h = O.solve_deterministic(ciphers[c], table, 120, seed, r)
            assert int(res.scores[j]) == s and res.history[j] == h
            assert np.array_equal(res.maps[j].astype(np.int64)[ciphers[c]], t)


def test_solve_with_restarts_deterministic_fold_and_stop(golden):
    cipher, table, seed, _, iters, _, _, _ = golden.det_run_cases()[0]
    cfg = cc.MasSolverConfig(mode="deterministic", workers=325, iterations=iters,
                             global_seed=seed, restarts=4)
    best, summ = cc.solve_with_restarts(cipher, cc.BigramTable(table), cfg)
    want = [O.solve_deterministic(cipher, table, iters, seed, r)[1] for r in range(4)]
    assert [s.score for s in summ] == want
    assert best.best_score == max(want) and best.restart_index == want.index(max(want))
    best2, summ2 = cc.solve_with_restarts(cipher, cc.BigramTable(table), cfg,
                                          stop=lambda res: res.restart_index == 1)
    assert len(summ2) == 2


# ------------------------------------------------------------------ n-gram extension (orders 2-4)
def test_ngram_kernel_order2_matches_reference_workers(golden):
    # the position-based n-gram kernel at order 2 must reproduce the reference's own
    # stochastic_worker outputs (tables fit uint16)
    cases = [c for c in golden.mas_worker_cases(O.permutation) if c[1].max() <= 65535]
    assert len(cases) >= 20
    for cipher, table, climb, seed, stream, want_text, want_score in cases:
        res = engine.mas_climb([cipher], [0], [philox_key(seed, stream)], table, climb,
                               ngram_kernel=True)
        assert int(res.scores[0]) == want_score
        assert np.array_equal(res.keys[0].astype(np.int64)[cipher], want_text)


def _ngram_cases(rng, order, n_cases=40):
    ciphers = []
    for i in range(n_cases):
        L = int(rng.choice([0, 1, order - 1, order, order + 1, 5, 17, 60, 100, 333, 600, 4096]))
        ciphers.append(rng.integers(0, int(rng.choice([3, 8, 26])), L))
    return ciphers


@pytest.mark.parametrize("order", [2, 3, 4])
def test_ngram_climb_vs_oracle(order):
    rng = np.random.default_rng(100 + order)
    ciphers = _ngram_cases(rng, order)
    for table in (rng.integers(0, 65536, 26**order), rng.integers(0, 50, 26**order)):
        seeds = [int(rng.integers(0, 2**63)) for _ in ciphers]
        streams = [int(rng.integers(0, 2**40)) for _ in ciphers]
        keys = np.array([philox_key(s, w) for s, w in zip(seeds, streams)], dtype=np.uint64)
        res = engine.mas_climb(ciphers, np.arange(len(ciphers)), keys, table, 1500, order=order,
                               draws_used=True, last_accept=True)
        want_s, want_m = O.ngram_workers(ciphers, np.arange(len(ciphers)), seeds, streams, order,
                                         table, 1500)
        assert res.scores.tolist() == want_s.tolist()
        for i, c in enumerate(ciphers):
            assert np.array_equal(res.keys[i].astype(np.int64)[c], want_m[i][c]), i


def test_ngram_climb_english_quadgram_and_early_exit(golden):
    corpus = "".join(chr(97 + int(x)) for x in golden.corpus())
    q4 = cc.quantize_log_table(cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus, 4)))
    rng = np.random.default_rng(5)
    plain = golden.plain_mas(471)
    ciphers = []
    for L in (60, 80, 100, 300, 471):
        key = rng.permutation(26)
        ciphers.append(key[plain[:L]])
    cof = np.repeat(np.arange(len(ciphers), dtype=np.int32), 8)
    seeds = [4242] * cof.size
    streams = list(range(cof.size))
    keys = philox_keys([4242], streams)
    full = engine.mas_climb(ciphers, cof, keys, q4.scores, 6000, order=4, group_size=8,
                            tries_done=True, computed=True)
    # most tries are served by the delta cache once the climb has settled
    assert (full.computed > 0).all() and full.computed.sum() < 0.5 * full.tries_done.sum()
    want_s, _ = O.ngram_workers(ciphers, cof, seeds, streams, 4, q4.scores, 6000)
    assert full.scores.tolist() == want_s.tolist()
    early = engine.mas_climb(ciphers, cof, keys, q4.scores, 6000, order=4, group_size=8,
                             tries_done=True, early_exit=True)
    assert early.scores.tolist() == full.scores.tolist()   # the early exit is exact
    assert np.array_equal(early.keys, full.keys)
    assert (early.tries_done <= 6000).all() and early.tries_done.min() < 6000
    assert early.group_best.tolist() == [int(np.argmax(want_s[i:i + 8])) for i in range(0, cof.size, 8)]


def test_ngram_skips_continue_the_stream():
    rng = np.random.default_rng(8)
    table = rng.integers(0, 1000, 26**3)
    c = rng.integers(0, 26, 150)
    key = philox_key(77, 3)
    a = engine.mas_climb([c], [0], [key], table, 700, order=3, draws_used=True)
    _, s_o, _, _ = O.ngram_worker(c, 3, table, 700, 77, 3, skip=int(a.draws_used[0]))
    b = engine.mas_climb([c], [0], [key], table, 700, order=3, skips=a.draws_used)
    assert int(b.scores[0]) == s_o


@pytest.mark.parametrize("order", [2, 3, 4])
def test_ngram_score_batch_vs_oracle(order):
    rng = np.random.default_rng(order)
    table = rng.integers(0, 2**40, 26**order)
    texts = [rng.integers(0, 26, int(L)) for L in rng.integers(0, 3000, 50)] + [np.zeros(0, int)]
    got = cc.ngram_score_text_batch(texts, cc.NgramTable(order, table))
    assert got.tolist() == [O.ngram_score_text(t, order, table) for t in texts]


def test_solve_stochastic_with_trigram_table():
    rng = np.random.default_rng(12)
    table = cc.NgramTable(3, rng.integers(0, 3000, 26**3))
    cipher = rng.integers(0, 26, 250)
    cfg = cc.MasSolverConfig(workers=16, climbings=3000, global_seed=99, restarts=2)
    best, summ = cc.solve_with_restarts(cipher, table, cfg)
    for r in range(2):
        want, _ = O.ngram_workers([cipher], np.zeros(16, np.int32), [99] * 16,
                                  [(r << 32) | w for w in range(16)], 3, table.scores, 3000)
        assert summ[r].score == int(want.max())
    assert best.best_score == cc.ngram_score_text(best.best_text, table)


@pytest.mark.parametrize("order", [2, 3, 4])
def test_ngram_log_score_bit_exact_vs_oracle(order):
    rng = np.random.default_rng(20 + order)
    logs = -rng.random(26**order) * 20 - 1
    lengths = [0, 1, order - 1, order, order + 1, 7, 8, 9, 127, 128, 129, 130, 400, 1000, 4096,
               4100, 9000]
    texts = [rng.integers(0, 26, L) for L in lengths]
    got = cc.ngram_log_score_text_batch(texts, cc.LogNgramTable(order, logs, -21.0))
    assert got.tolist() == [O.ngram_log_score_text(t, order, logs) for t in texts]


@pytest.mark.parametrize("order", [3, 4])
def test_sct_score_ngram_vs_oracle(order):
    rng = np.random.default_rng(30 + order)
    logs = -rng.random(26**order) * 20 - 1
    ciphers, keys, cof = [], [], []
    for i, (k, n) in enumerate([(5, 400), (10, 400), (20, 400), (7, 129), (40, 4096), (9, 5000)]):
        ciphers.append(rng.integers(0, 26, n))
        keys.append(rng.permutation(k))
    for i, (c, kk) in enumerate(zip(ciphers, keys)):
        got = engine.sct_score_batch([c], [0], kk[None, :].astype(np.uint8), logs, order=order)
        assert float(got[0]) == O.sct_score(c, logs, kk, order=order)


@pytest.mark.parametrize("order", [3, 4])
def test_sct_climb_ngram_vs_oracle(order):
    rng = np.random.default_rng(40 + order)
    corpus = rng.integers(0, 26, 5000)
    for k, n in [(5, 400), (10, 400), (20, 400), (15, 596), (33, 200), (6, order + 5)]:
        logs = -rng.random(26**order) * 20 - 1
        cipher = rng.integers(0, 26, n)
        seeds, streams = [int(rng.integers(0, 2**63))] * 6, list(range(6))
        keys = philox_keys(seeds[:1], streams)
        res = engine.sct_climb([cipher], np.zeros(6, np.int32), keys, logs, k, 1200, order=order,
                               group_size=6)
        want_s, want_k = O.sct_workers([cipher], np.zeros(6, np.int32), seeds, streams, logs, k,
                                       1200, order=order)
        assert res.scores.tolist() == want_s.tolist(), (k, n)
        assert np.array_equal(res.keys.astype(np.int64), want_k)


def test_solve_sct_trigram_recovers_key(golden):
    corpus = "".join(chr(97 + int(x)) for x in golden.corpus())
    l3 = cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus, 3))
    plain = golden.plain_sct(400)
    key = cc.WorkerRng(1234, cc.KEYGEN_STREAM).permutation(8)
    cipher = cc.sct_encrypt(plain, key)
    cfg = cc.SctSolverConfig(key_length=8, workers=64, climbings=4000, global_seed=5)
    best, _ = cc.solve_sct(cipher, l3, cfg)
    assert np.array_equal(best.best_text, plain)
    want_s, _ = O.sct_workers([cipher], np.zeros(64, np.int32), [5] * 64, list(range(64)), l3.logs,
                              8, 4000, order=3)
    assert best.per_worker_scores == want_s.tolist()


# ------------------------------------------------------------------ MAS kernel variants
@pytest.mark.parametrize("early", [False, True])
def test_mas_kernels_agree_with_oracle(early):
    # the D-form (maintained delta table), T-form and packed count-matrix kernels must give
    # the same per-worker outputs, equal to the oracle's stochastic_worker
    rng = np.random.default_rng(77 + early)
    ciphers = []
    for L in [2, 3, 5, 26, 60, 100, 300, 471, 1000, 2000]:
        c = rng.integers(0, int(rng.choice([2, 5, 26])), L)
        ciphers.append(c)
    table = rng.integers(0, 1000, 676)
    cof = np.repeat(np.arange(len(ciphers), dtype=np.int32), 6)
    streams = [int(rng.integers(0, 2**40)) for _ in cof]
    keys = philox_keys([2024], streams)
    outs = {}
    for kern in ("dform", "dtable", "tform", "packed"):
        outs[kern] = engine.mas_climb(ciphers, cof, keys, table, 5000, kernel=kern, draws_used=True,
                                      last_accept=True, tries_done=True, early_exit=early,
                                      group_size=6, accepts=True)
    want_s, want_m = O.mas_workers(ciphers, cof, [2024] * cof.size, streams, table, 5000)
    for kern, r in outs.items():
        assert r.scores.tolist() == want_s.tolist(), kern
        for i, c in enumerate(cof):
            assert np.array_equal(r.keys[i].astype(np.int64)[ciphers[c]], want_m[i][ciphers[c]]), kern
        # the early-exit point is kernel-specific (each stops once it has proven that no
        # proposal can be accepted); everything the reference defines must agree
        fields = ("last_accept", "group_best", "accepts") if early else (
            "draws_used", "last_accept", "tries_done", "group_best", "accepts")
        for f in fields:
            assert np.array_equal(getattr(r, f), getattr(outs["packed"], f)), (kern, f)
    if not early:
        assert (outs["dform"].tries_done == 5000).all()


def test_dform_draw_position_continues_stream():
    rng = np.random.default_rng(3)
    table = rng.integers(0, 700, 676)
    c = rng.integers(0, 26, 333)
    key = philox_key(5, 17)
    a = engine.mas_climb([c], [0], [key], table, 2345, kernel="dform", draws_used=True)
    b = engine.mas_climb([c], [0], [key], table, 777, kernel="dform", skips=a.draws_used)
    _, s_o, _, _ = O.stochastic_worker(c, table, 777, 5, 17, skip=int(a.draws_used[0]))
    assert int(b.scores[0]) == s_o
    assert int(a.draws_used[0]) == int(engine.mas_climb([c], [0], [key], table, 2345, kernel="packed",
                                                        draws_used=True).draws_used[0])


def test_packed_batch_and_out_buffers_match_list_api():
    from paper_2103_13937_b200 import _lib

    rng = np.random.default_rng(9)
    ciphers = [rng.integers(0, 26, int(L)) for L in rng.integers(2, 400, 30)]
    table = rng.integers(0, 800, 676)
    cof = np.repeat(np.arange(30, dtype=np.int32), 4)
    keys = philox_keys([3], list(range(cof.size)))
    want = engine.mas_climb(ciphers, cof, keys, table, 3000, group_size=4)
    out = engine.ClimbResult(scores=np.zeros(cof.size, np.int64), keys=np.zeros((cof.size, 26), np.uint8),
                             group_best=np.zeros(30, np.int64), draws_used=None, last_accept=None,
                             tries_done=None, launches=0)
    got = engine.mas_climb(_lib.Packed.of(ciphers), cof, keys, table, 3000, group_size=4, out=out)
    assert got is out
    assert np.array_equal(out.scores, want.scores) and np.array_equal(out.keys, want.keys)
    assert np.array_equal(out.group_best, want.group_best)
    with pytest.raises(ValueError):
        _lib.Packed(np.array([1, 2, 30], np.uint8), np.array([0, 3]))


@pytest.mark.parametrize("order", [2, 3])
def test_sct_ragged_key_lengths_one_launch(order):
    rng = np.random.default_rng(60 + order)
    logs = -rng.random(26**order) * 20 - 1
    ciphers = [rng.integers(0, 26, 400) for _ in range(12)]
    ks = [5, 6, 7, 9, 10, 12, 15, 17, 20, 33, 40, 64]
    cof = np.repeat(np.arange(12, dtype=np.int32), 3)
    klens = np.repeat(np.array(ks, dtype=np.int32), 3)
    streams = list(range(cof.size))
    keys = philox_keys([77], streams)
    res = engine.sct_climb(ciphers, cof, keys, logs, klens, 600, order=order, group_size=3,
                           draws_used=True)
    for i in range(cof.size):
        c, k = int(cof[i]), int(klens[i])
        key, score, _ = O.sct_worker(ciphers[c], logs, k, 600, 77, streams[i], order=order)
        assert float(res.scores[i]) == score, (i, k)
        assert np.array_equal(res.keys[i, :k].astype(np.int64), key)
    one = engine.sct_climb([ciphers[3]], np.zeros(3, np.int32), keys[9:12], logs, 9, 600, order=order,
                           draws_used=True)
    assert np.array_equal(one.scores, res.scores[9:12])
    assert np.array_equal(one.draws_used, res.draws_used[9:12])


@pytest.mark.parametrize("L,tmax", [(5000, 32_767), (40_000, 700), (3000, 100_000)])
def test_mas_kernel_gates_fall_back_exactly(L, tmax):
    """Inputs past the D-form gate ((n-1) max S >= 2^27), the T-form gate (n > 32768) and the
    16-bit table gate (max S > 65535) take the next kernel; results equal the oracle."""
    rng = np.random.default_rng(L)
    c = rng.integers(0, 26, L)
    table = rng.integers(0, tmax + 1, 676)
    table[7] = tmax
    keys = philox_keys([1], [0, 1])
    res = engine.mas_climb([c], np.zeros(2, np.int32), keys, table, 1200, draws_used=True)
    want_s, want_m = O.mas_workers([c], np.zeros(2, np.int32), [1, 1], [0, 1], table, 1200)
    assert res.scores.tolist() == want_s.tolist()
    assert np.array_equal(res.keys.astype(np.int64), want_m)


# ------------------------------------------------------------------ device-side test sets
def test_encrypt_batch_reference_recipe(golden):
    """WorkerRng(seed, KEYGEN).permutation(k) keys and mas/sct encryption on the GPU equal
    the host functions (pinned to the reference) for a ragged batch."""
    corpus = golden.corpus()
    rng = np.random.default_rng(5)
    lengths = [0, 1, 3, 26, 100, 400, 501] + [int(v) for v in rng.integers(2, 600, 25)]
    plains = [corpus[o:o + L] for o, L in zip(rng.integers(0, corpus.size - 700, len(lengths)), lengths)]
    seeds = [100000 + i for i in range(len(plains))]
    c_mas, k_mas = cc.encrypt_batch(plains, "mas", key_seeds=seeds)
    for p, s, c, k in zip(plains, seeds, c_mas, k_mas):
        want_k = O.permutation(s, 2**32 - 2, 26)
        assert np.array_equal(k, want_k)
        assert np.array_equal(c, cc.mas_encrypt(p, want_k))
    klens = [int(v) for v in rng.integers(1, 65, len(plains))]
    c_sct, k_sct = cc.encrypt_batch(plains, "sct", key_seeds=seeds, key_lengths=klens)
    for p, s, kl, c, k in zip(plains, seeds, klens, c_sct, k_sct):
        want_k = O.permutation(s, 2**32 - 2, kl)
        assert np.array_equal(k, want_k)
        assert np.array_equal(c, cc.sct_encrypt(p, want_k))
    # explicit keys
    keys = [rng.permutation(26) for _ in plains]
    c2, _ = cc.encrypt_batch(plains, "mas", keys=keys)
    assert all(np.array_equal(c, cc.mas_encrypt(p, k)) for p, c, k in zip(plains, c2, keys))
    with pytest.raises(ValueError):
        cc.encrypt_batch(plains[:1], "mas", keys=[np.zeros(26, int)])


# ------------------------------------------------------------------ randomized parity sweeps
def test_fuzz_mas_kernels_vs_oracle():
    """3,000 random workers: lengths 2..3000, alphabets of 2..26 letters, tables of many
    magnitudes (including the D-form / T-form gate edges), random budgets and stream skips."""
    rng = np.random.default_rng(2024)
    for trial in range(16):
        tmax = int(rng.choice([1, 5, 700, 32_767, 65_535, 2**20]))
        table = rng.integers(0, tmax + 1, 676)
        ciphers = []
        for _ in range(60):
            L = int(rng.choice([2, 3, 10, 100, 500, 1500, 3000]))
            ciphers.append(rng.integers(0, int(rng.integers(2, 27)), L))
        n = 500
        cof = rng.integers(0, len(ciphers), n).astype(np.int32)
        seeds = rng.integers(0, 2**63, n).tolist()
        streams = rng.integers(0, 2**48, n).tolist()
        keys = philox_keys(seeds, streams)
        climb = int(rng.choice([1, 33, 1000, 3000]))
        res = engine.mas_climb(ciphers, cof, keys, table, climb, last_accept=True)
        want_s, want_m = O.mas_workers(ciphers, cof, seeds, streams, table, climb)
        assert res.scores.tolist() == want_s.tolist(), (trial, tmax, climb)
        assert np.array_equal(res.keys.astype(np.int64), want_m), (trial, tmax, climb)


@pytest.mark.parametrize("order", [3, 4])
def test_fuzz_ngram_vs_oracle(order):
    rng = np.random.default_rng(300 + order)
    for trial in range(6):
        table = rng.integers(0, int(rng.choice([2, 300, 65_536])), 26**order)
        ciphers = [rng.integers(0, int(rng.integers(2, 27)), int(rng.choice([2, 5, 40, 90, 300, 1000])))
                   for _ in range(40)]
        n = 300
        cof = rng.integers(0, len(ciphers), n).astype(np.int32)
        seeds = rng.integers(0, 2**63, n).tolist()
        streams = rng.integers(0, 2**48, n).tolist()
        keys = philox_keys(seeds, streams)
        res = engine.mas_climb(ciphers, cof, keys, table, 800, order=order)
        want_s, _ = O.ngram_workers(ciphers, cof, seeds, streams, order, table, 800)
        assert res.scores.tolist() == want_s.tolist(), trial


def test_fuzz_sct_vs_oracle():
    rng = np.random.default_rng(77)
    for trial in range(10):
        n = int(rng.choice([8, 129, 400, 1000]))
        logs = -rng.random(676) * 20 - 1
        ciphers = [rng.integers(0, 26, n) for _ in range(4)]
        m = 64
        cof = rng.integers(0, 4, m).astype(np.int32)
        klens = rng.integers(2, min(n, 64) + 1, m).astype(np.int32)
        seeds = rng.integers(0, 2**63, m).tolist()
        streams = rng.integers(0, 2**48, m).tolist()
        keys = philox_keys(seeds, streams)
        p1, p2 = sorted(int(v) for v in rng.integers(0, 101, 2))
        res = engine.sct_climb(ciphers, cof, keys, logs, klens, 300, p1=p1, p2=p2, op1_hop=2,
                               op2_hop=4)
        for i in range(m):
            k = int(klens[i])
            key, score, _ = O.sct_worker(ciphers[cof[i]], logs, k, 300, seeds[i], streams[i],
                                         p1=p1, p2=p2, op1_hop=2, op2_hop=4)
            assert float(res.scores[i]) == score, (trial, i)
            assert np.array_equal(res.keys[i, :k].astype(np.int64), key)


def test_batch_solvers_equal_per_ciphertext_solves(golden):
    rng = np.random.default_rng(21)
    table = cc.BigramTable(golden.english_scores())
    ciphers = [rng.integers(0, 26, int(L)) for L in (50, 120, 300)]
    cfg = cc.MasSolverConfig(workers=16, climbings=3000, global_seed=5)
    got = cc.solve_stochastic_batch(ciphers, table, cfg, restart=2, seeds=[5, 6, 7])
    for c, s, g in zip(ciphers, (5, 6, 7), got):
        want = cc.solve_stochastic(c, table, cc.MasSolverConfig(workers=16, climbings=3000,
                                                                 global_seed=s), restart=2)
        assert g.per_worker_scores == want.per_worker_scores
        assert np.array_equal(g.best_text, want.best_text)
    logs = cc.LogBigramTable(golden.english_logs(), -24.0)
    sct_c = [rng.integers(0, 26, 240) for _ in range(3)]
    scfg = cc.SctSolverConfig(key_length=6, workers=8, climbings=600, global_seed=9)
    got = cc.solve_sct_batch(sct_c, logs, scfg, key_lengths=[5, 6, 9])
    for c, k, g in zip(sct_c, (5, 6, 9), got):
        want, _ = cc.solve_sct(c, logs, cc.SctSolverConfig(key_length=k, workers=8, climbings=600,
                                                           global_seed=9))
        assert g.per_worker_scores == want.per_worker_scores
        assert np.array_equal(g.best_key, want.best_key)


def test_worker_tickets_with_more_workers_than_resident_warps():
    """Batches larger than the resident grid hand out workers through the ticket counter
    (ccg_internal.h WorkerTickets): sampled workers of the D-form, n-gram and SCT warp
    kernels still equal the oracle."""
    rng = np.random.default_rng(404)
    n = 12_000
    sample = rng.choice(n, 48, replace=False)
    cs = [rng.integers(0, 26, int(L)) for L in rng.integers(30, 200, 50)]
    cof = rng.integers(0, len(cs), n).astype(np.int32)
    seeds = [int(v) for v in rng.integers(0, 2**63, n)]
    streams = [int(v) for v in rng.integers(0, 2**40, n)]
    keys = philox_keys(seeds, streams)
    table = rng.integers(0, 900, 676)
    res = engine.mas_climb(cs, cof, keys, table, 300)
    s, _ = O.mas_workers(cs, cof[sample], [seeds[i] for i in sample],
                         [streams[i] for i in sample], table, 300)
    assert res.scores[sample].tolist() == s.tolist()
    t3 = rng.integers(0, 60000, 26**3)
    res = engine.mas_climb(cs, cof, keys, t3, 200, order=3)
    s, _ = O.ngram_workers(cs, cof[sample], [seeds[i] for i in sample],
                           [streams[i] for i in sample], 3, t3, 200)
    assert res.scores[sample].tolist() == s.tolist()
    sc = [rng.integers(0, 26, 150) for _ in range(4)]
    scof = rng.integers(0, 4, n).astype(np.int32)
    logs = -rng.random(676) * 20 - 1
    res = engine.sct_climb(sc, scof, keys, logs, 9, 40)
    for i in sample[:16]:
        _, want, _ = O.sct_worker(sc[scof[i]], logs, 9, 40, seeds[i], streams[i])
        assert float(res.scores[i]) == want


def test_ngram_lookups_counter_and_l2_microbench():
    """The n-gram climb's table-read counter (the C4 roofline numerator) is consistent with its
    walk counter, does not change any result, and the L2 gather microbenchmark runs."""
    rng = np.random.default_rng(4040)
    table = rng.integers(0, 65536, 26**4)
    cs = [rng.integers(0, 26, int(L)) for L in (60, 80, 100)]
    cof = np.repeat(np.arange(3, dtype=np.int32), 64)
    keys = philox_keys([9], list(range(cof.size)))
    a = engine.mas_climb(cs, cof, keys, table, 2000, order=4, computed=True, lookups=True)
    b = engine.mas_climb(cs, cof, keys, table, 2000, order=4)
    assert np.array_equal(a.scores, b.scores) and np.array_equal(a.keys, b.keys)
    assert (a.lookups >= 4 * a.computed).all() and a.lookups.sum() > 0
    assert engine.bench_l2_gather(26**4) > 1e10
