"""GPU parity of the one-worker-per-lane SCT kernels (csrc/ccg_sct_lane.cu) through the C ABI.

Parity mode (the default throughput path of ccg_sct_climb): every per-worker output --
float64 score (numpy pairwise order), key, draws consumed, last accepted try -- must equal the
oracle's sct_worker (oracle/cc_oracle.c, pinned to the reference by tests/test_oracle_golden.py)
and the warp / speculative kernels' bit for bit.

Fast mode (opt-in, ccg_sct_fast_climb): the quantised integer fitness with incremental
rescoring must equal its own oracle (cco_sct_fast_worker, full rescore) bit for bit, and on a
dyadic log table -- where the quantisation is exact and every float64 sum is exact too -- it
must reproduce the reference algorithm's climb key for key.
"""
import numpy as np
import pytest

import paper_2103_13937_b200 as cc
from paper_2103_13937_b200 import engine
from paper_2103_13937_b200.rng import philox_keys
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    from paper_2103_13937_b200 import _lib

    if _lib.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def _oracle_parity(ciphers, cof, klens, seed, streams, logs, climbings, order, **kw):
    """Per-worker oracle outputs for a ragged batch (the oracle's batch API takes one k)."""
    n = len(cof)
    scores = np.empty(n)
    keys = [None] * n
    last = np.empty(n, np.int64)
    for i in range(n):
        k, sc, la = O.sct_worker(ciphers[cof[i]], logs, int(klens[i]), climbings, seed,
                                 streams[i], order=order, **kw)
        keys[i], scores[i], last[i] = k, sc, la
    return scores, keys, last


@pytest.mark.parametrize("order", [2, 3])
def test_lane_kernel_every_short_key_length(order):
    """Every key length 2..20 (and 31, 32) on short texts: an 8-position letter block wraps
    several rows when k < 8 and exactly one row end for k >= 8 -- the extended colstart
    (cs[m] = cs[m mod k] + m div k) must give the same letters as the per-position walk."""
    rng = np.random.default_rng(900 + order)
    logs = -rng.random(26**order) * 20 - 1
    ks = list(range(2, 21)) + [31, 32]
    ciphers = [rng.integers(0, 26, L) for L in (41, 64, 97)]
    cof = np.array([i % 3 for i in range(len(ks) * 4)], np.int32)
    klens = np.array([ks[i // 4] for i in range(len(cof))], np.int32)
    streams = [int(s) for s in rng.integers(0, 2**40, len(cof))]
    keys = philox_keys([77], streams)
    res = engine.sct_climb(ciphers, cof, keys, logs, klens, 300, order=order, kernel="lane")
    want_s, want_k, _ = _oracle_parity(ciphers, cof, klens, 77, streams, logs, 300, order)
    assert res.scores.tolist() == want_s.tolist()
    for i in range(len(cof)):
        assert np.array_equal(res.keys[i, :klens[i]].astype(np.int64), want_k[i]), i


@pytest.mark.parametrize("order", [2, 3, 4])
def test_lane_kernel_vs_oracle(order):
    """Ragged text lengths AND key lengths in one launch, chunks of 32 workers spanning
    several ciphertexts (extra passes), keys up to 64 positions (the wide variant)."""
    rng = np.random.default_rng(500 + order)
    logs = -rng.random(26**order) * 20 - 1
    lens = [400, 137, 596, 64, 400, 9, 1000, 251]
    ciphers = [rng.integers(0, 26, L) for L in lens]
    m = 70
    cof = rng.integers(0, len(ciphers), m).astype(np.int32)
    cof[:32] = 0  # one full chunk of one ciphertext
    klens = np.array([int(rng.integers(2, min(64, lens[c]) + 1)) for c in cof], np.int32)
    klens[5] = min(64, lens[cof[5]])
    streams = [int(s) for s in rng.integers(0, 2**40, m)]
    seed = 4242
    keys = philox_keys([seed], streams)
    for climb in (0, 1, 377):
        res = engine.sct_climb(ciphers, cof, keys, logs, klens, climb, order=order, kernel="lane",
                               draws_used=True, last_accept=True, tries_done=True)
        want_s, want_k, want_last = _oracle_parity(ciphers, cof, klens, seed, streams, logs, climb,
                                                   order)
        assert res.scores.tolist() == want_s.tolist(), climb
        for i in range(m):
            assert np.array_equal(res.keys[i, :klens[i]].astype(np.int64), want_k[i]), (climb, i)
        assert np.array_equal(res.last_accept, want_last), climb
        assert (res.tries_done == climb).all()


@pytest.mark.parametrize("order,kmax", [(2, 20), (3, 40), (4, 12)])
def test_lane_warp_and_speculative_kernels_agree(order, kmax):
    """All three SCT kernels give identical per-worker outputs, draws consumed included."""
    rng = np.random.default_rng(600 + order)
    logs = -rng.random(26**order) * 20 - 1
    cs = [rng.integers(0, 26, 333) for _ in range(3)]
    m = 96
    cof = np.repeat(np.arange(3, dtype=np.int32), 32)
    klens = rng.integers(2, kmax + 1, m).astype(np.int32)
    keys = philox_keys([99], list(range(m)))
    kw = dict(order=order, draws_used=True, last_accept=True, tries_done=True)
    lane = engine.sct_climb(cs, cof, keys, logs, klens, 700, kernel="lane", **kw)
    warp = engine.sct_climb(cs, cof, keys, logs, klens, 700, kernel="warp", speculate=False, **kw)
    spec = engine.sct_climb(cs, cof, keys, logs, klens, 700, kernel="warp", **kw)
    for other in (warp, spec):
        assert lane.scores.tolist() == other.scores.tolist()
        assert np.array_equal(lane.keys, other.keys)
        assert np.array_equal(lane.draws_used, other.draws_used)
        assert np.array_equal(lane.last_accept, other.last_accept)


def test_lane_kernel_skips_and_trigram_table_in_l2():
    rng = np.random.default_rng(77)
    logs = -rng.random(26**3) * 20 - 1
    cipher = rng.integers(0, 26, 400)
    m = 40
    keys = philox_keys([5], list(range(m)))
    skips = rng.integers(0, 50, m).astype(np.uint64)
    a = engine.sct_climb([cipher], np.zeros(m, np.int32), keys, logs, 13, 500, order=3,
                         kernel="lane", skips=skips, draws_used=True)
    b = engine.sct_climb([cipher], np.zeros(m, np.int32), keys, logs, 13, 500, order=3,
                         kernel="lane", skips=skips, draws_used=True, table_l2=True)
    assert np.array_equal(a.scores, b.scores) and np.array_equal(a.keys, b.keys)
    for i in (0, 7, 39):
        k, s, _ = O.sct_worker(cipher, logs, 13, 500, 5, i, skip=int(skips[i]), order=3)
        assert float(a.scores[i]) == s and np.array_equal(a.keys[i].astype(np.int64), k)


def test_lane_kernel_golden_acceptance_08(golden):
    """The reference's own solve_sct output for acceptance #08's input (64 workers x 15,000,
    frozen in tests/golden) reproduced by the lane kernel, worker by worker."""
    g = golden.load("sct_solve")
    cipher = g["cipher"].astype(np.int64)
    keys = philox_keys([8000], list(range(64)))
    res = engine.sct_climb([cipher], np.zeros(64, np.int32), keys, golden.english_logs(), 10,
                           15_000, kernel="lane", group_size=64)
    assert res.scores.tolist() == g["per_worker"].tolist()
    assert np.array_equal(res.keys[int(res.group_best[0])], g["best_key"])


# ------------------------------------------------------------------ fast mode
def _fast_oracle(ciphers, cof, klens, seed, streams, q, order, climbings):
    n = len(cof)
    scores = np.empty(n, np.int64)
    keys = [None] * n
    for i in range(n):
        k, s, _ = O.sct_fast_worker(ciphers[cof[i]], q, order, int(klens[i]), climbings, seed,
                                    streams[i])
        keys[i], scores[i] = k, s
    return scores, keys


@pytest.mark.parametrize("order", [2, 3, 4])
def test_fast_mode_vs_its_oracle(order):
    rng = np.random.default_rng(700 + order)
    lt = cc.LogNgramTable(order, -rng.random(26**order) * 20 - 1, -24.0) if order > 2 else \
        cc.LogBigramTable(-rng.random(676) * 20 - 1, -24.0)
    q = cc.quantize_sct_table(lt, text_len=1000)
    lens = [400, 137, 596, 1000, 33]
    ciphers = [rng.integers(0, 26, L) for L in lens]
    m = 80
    cof = rng.integers(0, len(ciphers), m).astype(np.int32)
    cof[:32] = 2
    klens = np.array([int(rng.integers(2, min(64, lens[c]) + 1)) for c in cof], np.int32)
    streams = list(range(m))
    keys = philox_keys([31], streams)
    for climb in (0, 250):
        res = engine.sct_fast_climb(ciphers, cof, keys, q, klens, climb, group_size=0,
                                    last_accept=True, draws_used=True)
        want_s, want_k = _fast_oracle(ciphers, cof, klens, 31, streams, q.table, order, climb)
        assert res.scores.tolist() == want_s.tolist(), climb
        for i in range(m):
            assert np.array_equal(res.keys[i, :klens[i]].astype(np.int64), want_k[i]), (climb, i)
        # the same stream positions as the parity climb (identical proposals)
        par = engine.sct_climb(ciphers, cof, keys, lt.logs, klens, climb, order=order,
                               kernel="lane", draws_used=True)
        assert np.array_equal(res.draws_used, par.draws_used)
        if climb:
            full = np.array([len(ciphers[c]) - order + 1 for c in cof]) * climb
            assert (res.lookups > 0).all() and (res.lookups <= full).all()


@pytest.mark.parametrize("order", [2, 3])
def test_fast_mode_window_tables_on_regular_grids(order):
    """Regular grids (text length a multiple of k) read the changed windows from the
    per-(ciphertext, k) window-sum tables (ccg_sct_lane.cu sct_ftab_kernel): identical to the
    fast mode's oracle and to the column walk, with one table read per changed window."""
    rng = np.random.default_rng(720 + order)
    lt = cc.LogNgramTable(order, -rng.random(26**order) * 20 - 1, -24.0) if order > 2 else \
        cc.LogBigramTable(-rng.random(676) * 20 - 1, -24.0)
    q = cc.quantize_sct_table(lt, text_len=600)
    ciphers = [rng.integers(0, 26, L) for L in (400, 120, 600, 45)]
    pairs = [(0, k) for k in (order, 4, 5, 8, 10, 16, 20, 25, 40)] + \
            [(1, k) for k in (order, 6, 12, 15, 24, 30)] + [(2, k) for k in (12, 25, 30)] + \
            [(3, k) for k in (order, 5, 9, 15)] + [(0, 7), (1, 7)]  # (+ two irregular grids)
    pairs = [(c, k) for c, k in pairs if k >= order]
    cof = np.array([c for c, _ in pairs for _ in range(3)], np.int32)
    klens = np.array([k for _, k in pairs for _ in range(3)], np.int32)
    m = cof.size
    streams = list(range(m))
    keys = philox_keys([77], streams)
    for climb in (0, 300):
        res = engine.sct_fast_climb(ciphers, cof, keys, q, klens, climb, draws_used=True)
        walk = engine.sct_fast_climb(ciphers, cof, keys, q, klens, climb, draws_used=True,
                                     window_tables=False)
        want_s, want_k = _fast_oracle(ciphers, cof, klens, 77, streams, q.table, order, climb)
        assert res.scores.tolist() == want_s.tolist() == walk.scores.tolist(), climb
        for i in range(m):
            assert np.array_equal(res.keys[i, :klens[i]].astype(np.int64), want_k[i]), (climb, i)
        assert np.array_equal(res.draws_used, walk.draws_used)
        if climb:
            # tabulated: regular grid and order * k**order <= 2**17 entries (kSctFTabMaxEntries)
            regular = np.array([len(ciphers[c]) % k == 0 and order * int(k)**order <= 2**17
                                for c, k in zip(cof, klens)])
            assert (res.lookups[regular] <= walk.lookups[regular]).all()
            assert res.lookups[regular].sum() * 5 < walk.lookups[regular].sum()
            assert (res.lookups[~regular] == walk.lookups[~regular]).all()
            bad = [(int(c), int(k), int(v)) for c, k, v, r in zip(cof, klens, res.lookups, regular)
                   if r and v > k * climb]
            assert not bad, bad


@pytest.mark.parametrize("order", [2, 3])
def test_fast_mode_reduces_to_reference_climb_on_a_dyadic_table(order):
    """With log-probabilities that are multiples of 2^-10 (>= -24), quantising at shift 10 is
    exact and every float64 partial sum is exact, so the fast mode's integer fitness is the
    reference's float64 fitness times 2^10: both climbs take identical decisions."""
    rng = np.random.default_rng(800 + order)
    logs = -rng.integers(1, 24 * 1024, 26**order) / 1024.0
    lt = cc.LogNgramTable(order, logs, -24.0) if order > 2 else cc.LogBigramTable(logs, -24.0)
    q = cc.quantize_sct_table(lt, text_len=600, max_shift=10)
    assert q.shift == 10 and np.array_equal(q.table.astype(np.float64), logs * 1024)
    ciphers = [rng.integers(0, 26, 400), rng.integers(0, 26, 596)]
    cof = np.repeat(np.array([0, 1], np.int32), 32)
    klens = np.repeat(np.array([10, 15], np.int32), 32)
    keys = philox_keys([17], list(range(64)))
    fast = engine.sct_fast_climb(ciphers, cof, keys, q, klens, 2000, group_size=32)
    par = engine.sct_climb(ciphers, cof, keys, logs, klens, 2000, order=order, group_size=32)
    assert np.array_equal(fast.keys, par.keys)
    assert np.array_equal(fast.scores.astype(np.float64), par.scores * 1024)
    assert np.array_equal(fast.group_best, par.group_best)


def test_fast_mode_validates():
    lt = cc.LogBigramTable(np.full(676, -10.0), -24.0)
    q = cc.quantize_sct_table(lt, text_len=100)
    keys = philox_keys([1], [0])
    with pytest.raises(ValueError):
        engine.sct_fast_climb([np.zeros(5, np.int64)], [0], keys, q, 6, 10)  # shorter than key
    big = cc.QuantizedSctTable(2, np.full(676, -(2**30), np.int32), 30)
    with pytest.raises(cc.engine._lib.EngineError):
        engine.sct_fast_climb([np.zeros(50, np.int64)], [0], keys, big, 5, 10)  # int32 overflow


def test_lane_kernels_take_any_reference_hop_count():
    """op1_hop / op2_hop up to 3 (the reference default) run on the per-lane kernels
    (bit-exact); larger hop counts (valid for the reference, sct.py:57-66) take the warp
    kernel automatically, and the fast mode refuses them loudly."""
    rng = np.random.default_rng(901)
    logs = -rng.random(676) * 20 - 1
    cipher = rng.integers(0, 26, 300)
    keys = philox_keys([3], list(range(40)))
    for h1, h2 in [(3, 1), (1, 3), (2, 3)]:
        res = engine.sct_climb([cipher], np.zeros(40, np.int32), keys, logs, 17, 300, op1_hop=h1,
                               op2_hop=h2, kernel="lane")
        want, wk = O.sct_workers([cipher], np.zeros(40, np.int32), [3] * 40, list(range(40)), logs,
                                 17, 300, op1_hop=h1, op2_hop=h2)
        assert res.scores.tolist() == want.tolist()
        assert np.array_equal(res.keys.astype(np.int64), wk)
    res = engine.sct_climb([cipher], np.zeros(40, np.int32), keys, logs, 17, 300, op1_hop=9,
                           op2_hop=12)
    want, _ = O.sct_workers([cipher], np.zeros(40, np.int32), [3] * 40, list(range(40)), logs, 17,
                            300, op1_hop=9, op2_hop=12)
    assert res.scores.tolist() == want.tolist()
    q = cc.quantize_sct_table(cc.LogBigramTable(logs, -24.0), text_len=300)
    with pytest.raises(cc.engine._lib.EngineError):
        engine.sct_fast_climb([cipher], np.zeros(40, np.int32), keys, q, 17, 10, op1_hop=9)


def test_solve_sct_fast_public_api(golden):
    """solve_sct_fast: the reference's solve_sct restart loop in the fast mode, through the
    public API; recovers the acceptance #08 (k = 10) key and matches its oracle per worker."""
    plain = golden.plain_sct(596)
    logs = cc.LogBigramTable(golden.english_logs(), -24.0)
    cipher = cc.sct_encrypt(plain, O.permutation(800, golden.KEYGEN_STREAM, 10))
    cfg = cc.SctSolverConfig(key_length=10, workers=64, climbings=15_000, restarts=5,
                             global_seed=8000)
    best, runs = cc.solve_sct_fast(cipher, logs, cfg,
                                   stop=lambda r: bool(np.array_equal(r.best_text, plain)))
    assert np.array_equal(best.best_text, plain)
    q = cc.quantize_sct_table(logs, text_len=596)
    want, _ = O.sct_fast_workers([cipher], np.zeros(64, np.int32), [8000] * 64, list(range(64)),
                                 q.table, 2, 10, 15_000)
    first = cc.solve_sct_fast(cipher, logs, cc.SctSolverConfig(key_length=10, workers=64,
                                                               global_seed=8000))[0]
    assert [int(round(v * 2.0**q.shift)) for v in first.per_worker_scores] == want.tolist()


def test_compressed_trigram_tables(golden):
    """A trigram log table with few distinct entries (the corpus table: log2 of small counts)
    is held as a byte index + distinct values in shared memory; results are bit-identical to
    the table read through L2 and to the oracle, in both the parity and the fast mode."""
    corpus = "".join(chr(97 + int(x)) for x in golden.corpus())
    l3 = cc.build_log_ngram_table(cc.build_ngram_table_from_corpus(corpus, 3))
    assert np.unique(l3.logs).size <= 256
    rng = np.random.default_rng(77)
    ciphers = [rng.integers(0, 26, L) for L in (400, 251)]
    cof = np.repeat(np.array([0, 1], np.int32), 32)
    klens = np.repeat(np.array([13, 7], np.int32), 32)
    keys = philox_keys([12], list(range(64)))
    a = engine.sct_climb(ciphers, cof, keys, l3.logs, klens, 800, order=3, kernel="lane")
    b = engine.sct_climb(ciphers, cof, keys, l3.logs, klens, 800, order=3, kernel="lane",
                         table_l2=True)
    assert a.scores.tolist() == b.scores.tolist() and np.array_equal(a.keys, b.keys)
    for i in (0, 31, 32, 63):
        k, s, _ = O.sct_worker(ciphers[cof[i]], l3.logs, int(klens[i]), 800, 12, i, order=3)
        assert float(a.scores[i]) == s and np.array_equal(a.keys[i, :klens[i]].astype(np.int64), k)
    q = cc.quantize_sct_table(l3, text_len=400)
    fa = engine.sct_fast_climb(ciphers, cof, keys, q, klens, 800)
    fb = engine.sct_fast_climb(ciphers, cof, keys, q, klens, 800, table_l2=True)
    assert fa.scores.tolist() == fb.scores.tolist() and np.array_equal(fa.keys, fb.keys)
    for i in (0, 63):
        k, s, _ = O.sct_fast_worker(ciphers[cof[i]], q.table, 3, int(klens[i]), 800, 12, i)
        assert int(fa.scores[i]) == s


@pytest.mark.parametrize("order", [2, 3, 4])
def test_lane_kernels_tiny_texts(order):
    """Texts shorter than (or as long as) the n-gram order -- an empty or single-window
    pairwise sum -- in both modes, ragged in one launch."""
    rng = np.random.default_rng(1200 + order)
    logs = -rng.random(26**order) * 20 - 1
    ciphers = [rng.integers(0, 26, L) for L in (2, 3, 4, 5, 9)]
    cof = np.repeat(np.arange(5, dtype=np.int32), 8)
    klens = np.array([2 if len(ciphers[c]) < 4 else int(rng.integers(2, len(ciphers[c]) + 1))
                      for c in cof], np.int32)
    keys = philox_keys([21], list(range(cof.size)))
    res = engine.sct_climb(ciphers, cof, keys, logs, klens, 120, order=order, kernel="lane")
    lt = cc.LogNgramTable(order, logs, -30.0) if order > 2 else cc.LogBigramTable(logs, -30.0)
    q = cc.quantize_sct_table(lt, text_len=9)
    fres = engine.sct_fast_climb(ciphers, cof, keys, q, klens, 120)
    for i in range(cof.size):
        c, k = ciphers[cof[i]], int(klens[i])
        key, s, _ = O.sct_worker(c, logs, k, 120, 21, i, order=order)
        assert float(res.scores[i]) == s and np.array_equal(res.keys[i, :k].astype(np.int64), key)
        fkey, fs, _ = O.sct_fast_worker(c, q.table, order, k, 120, 21, i)
        assert int(fres.scores[i]) == fs and np.array_equal(fres.keys[i, :k].astype(np.int64), fkey)
