"""CPU-only checks: the C-ABI library loads and exports its header, the host layer's
reference semantics (key derivation, validation, table building, ciphers, restart fold),
and that the product path fails loudly without a GPU (no CPU fallback)."""
import re
import ctypes
import warnings
from pathlib import Path

import numpy as np
import pytest

import paper_2103_13937_b200 as cc
from paper_2103_13937_b200 import _lib, engine
from oracle import oracle as O

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "cipherclimb_b200.h").read_text()
    return sorted(set(re.findall(r"\b(ccg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 25
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.EXPORTS), set(syms) ^ set(_lib.EXPORTS)
    assert _lib.load().ccg_abi_version() == _lib.ABI_VERSION


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_lib.EngineError):
        cc.solve_stochastic(np.array([0, 1, 2, 1]), cc.BigramTable(np.ones(676, np.int64)),
                            cc.MasSolverConfig(workers=2, climbings=10))
    with pytest.raises(_lib.EngineError):
        cc.score_text(np.array([0, 1]), cc.BigramTable(np.ones(676, np.int64)))


def test_philox_key_matches_numpy_conversion():
    rng = np.random.default_rng(0)
    vals = [0, 1, 2**53 + 1, 2**63 - 1, 2**63, 2**63 + 1025, 2**64 - 1, 2**64 - 1025, -1, -7,
            (5 << 32) | 17, 2**32 - 2]
    vals += [int(x) for x in rng.integers(0, 2**63, 10, dtype=np.uint64)]
    for s in vals:
        for w in vals:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                k = np.asarray([s % 2**64, w % 2**64]).astype(np.uint64)
            assert cc.philox_key(s, w) == (int(k[0]), int(k[1])) == O.reference_key(s, w)


def test_stream_indices():
    assert cc.worker_stream_index(3, 7) == (3 << 32) | 7
    assert cc.pivot_stream_index(2) == (2 << 32) | (2**32 - 1)
    with pytest.raises(ValueError):
        cc.worker_stream_index(0, 2**32 - 2)
    with pytest.raises(ValueError):
        cc.worker_stream_index(-1, 0)
    assert cc.uniform_to_int(0.999, 26) == 25
    with pytest.raises(ValueError):
        cc.uniform_to_int(0.5, 0)


@pytest.mark.parametrize("n,shards,align", [(0, 3, 1), (1, 8, 1), (64, 8, 1), (100, 3, 1),
                                            (640, 8, 64), (130, 4, 64), (7, 2, 5)])
def test_shard_bounds(n, shards, align):
    b = engine.shard_bounds(n, shards, align)
    covered = [i for lo, hi in b for i in range(lo, hi)]
    assert covered == list(range(n))
    assert len(b) <= shards
    for lo, hi in b[:-1]:
        assert hi % align == 0
    if b:
        sizes = [hi - lo for lo, hi in b]
        assert max(sizes) - min(sizes) <= align


def test_configs_validate_like_reference():
    with pytest.raises(ValueError, match="unknown mode"):
        cc.MasSolverConfig(mode="x")
    with pytest.raises(ValueError, match="workers=325"):
        cc.MasSolverConfig(mode="deterministic", workers=64)
    with pytest.raises(ValueError, match="climbings must be at least 1"):
        cc.MasSolverConfig(climbings=0)
    with pytest.raises(ValueError, match="key_length"):
        cc.SctSolverConfig(key_length=1)
    with pytest.raises(ValueError, match="thresholds"):
        cc.SctSolverConfig(key_length=5, p1=70, p2=60)
    with pytest.raises(ValueError, match="non-negative"):
        cc.SctSolverConfig(key_length=5, climbings=-1)
    cc.SctSolverConfig(key_length=5, climbings=0)
    with pytest.raises(ValueError, match="two distinct letters"):
        cc.solve_stochastic(np.array([3, 3, 3]), cc.BigramTable(np.ones(676, np.int64)),
                            cc.MasSolverConfig())
    with pytest.raises(ValueError, match="shorter than the key"):
        cc.solve_sct(np.arange(5), cc.LogBigramTable(-np.ones(676), -2.0),
                     cc.SctSolverConfig(key_length=10))


def test_tables_from_corpus_match_reference(golden):
    eng = golden.english_scores()
    from paper_2103_13937_b200.codec import ALPHABET

    corpus_text = "".join(ALPHABET[i] for i in golden.corpus())
    t = cc.build_table_from_corpus(corpus_text)
    assert np.array_equal(t.scores, eng)
    logs = cc.build_log_table(t)
    assert logs.logs.tolist() == golden.english_logs().tolist()  # bit-exact
    text = cc.format_bigram_file(t)
    assert np.array_equal(cc.parse_bigram_file(text).scores, eng)
    with pytest.warns(UserWarning):
        cc.parse_bigram_file("ab 3\nab 4\n")
    for bad in ("ab", "abc 1", "aB 1", "ab x", "ab -1"):
        with pytest.raises(ValueError):
            cc.parse_bigram_file(bad)
    with pytest.raises(ValueError):
        cc.build_log_table(t, floor=-1.0)


def test_codec():
    assert cc.normalize("Always remember, that!") == "alwaysrememberthat"
    assert cc.demap(cc.map_text("hello")) == "hello"
    with pytest.raises(ValueError):
        cc.map_text("Hello")
    assert cc.demap(np.array([], dtype=np.int64)) == ""


def test_pairs():
    assert cc.index_to_pair(0) == (0, 1) and cc.index_to_pair(324) == (24, 25)
    t = 0
    for i in range(26):
        for j in range(i + 1, 26):
            assert cc.index_to_pair(t) == (i, j) and cc.pair_to_index(i, j) == t
            t += 1


def test_cipher_helpers_vs_oracle(golden):
    for key, n, want in golden.gather_cases(O.permutation):
        assert np.array_equal(cc.transposition_gather_map(key, n), want)
    rng = np.random.default_rng(5)
    for k in (2, 5, 10, 17):
        for n in (k, 3 * k + 1, 100):
            key = rng.permutation(k)
            t = rng.integers(0, 26, n)
            assert np.array_equal(cc.sct_decrypt(cc.sct_encrypt(t, key), key), t)
            assert np.array_equal(cc.sct_decrypt(t, key), O.sct_decrypt(t, key))
    mk = rng.permutation(26)
    t = rng.integers(0, 26, 50)
    assert np.array_equal(cc.mas_decrypt(cc.mas_encrypt(t, mk), mk), t)
    assert np.array_equal(cc.apply_letter_swap(np.array([0, 1, 2]), 0, 2), [2, 1, 0])


def test_select_operator():
    Op = cc.Operator
    assert cc.select_operator(10, 33, 66) is Op.ELEMENT_SWAP
    assert cc.select_operator(33, 33, 66) is Op.BLOCK_SWAP
    assert cc.select_operator(66, 33, 66) is Op.BLOCK_SHIFT
    with pytest.raises(ValueError):
        cc.select_operator(100, 33, 66)


def test_max_element_and_restart_fold():
    assert cc.max_element([4, 9, 9]) == (1, 9)
    with pytest.raises(ValueError):
        cc.max_element([])
    from paper_2103_13937_b200.search import run_restarts

    scores = [5, 7, 7, 3]

    def solve_one(r):
        return cc.SolveResult(np.array([r]), scores[r], [scores[r]], [])

    best, runs = run_restarts(solve_one, 4)
    assert best.restart_index == 1 and [r.restart for r in runs] == [0, 1, 2, 3]
    best, runs = run_restarts(solve_one, 4, stop=lambda r: r.best_score == 7)
    assert len(runs) == 2 and best.best_score == 7


def test_bench_workload_keys_match_oracle():
    import bench

    for s in (100000, 100001, 100777):
        assert np.array_equal(bench.reference_permutation(s, bench.KEYGEN_STREAM, 26),
                              O.permutation(s, bench.KEYGEN_STREAM, 26))


def test_ngram_file_formats_round_trip(golden):
    import paper_2103_13937_b200 as cc

    eng = cc.BigramTable(golden.english_scores())
    # order 2 is byte-identical to the reference's bigram format
    assert cc.format_ngram_file(eng) == cc.format_bigram_file(eng)
    assert np.array_equal(cc.parse_ngram_file(cc.format_bigram_file(eng), 2).scores, eng.scores)
    corpus = "".join(chr(97 + int(x)) for x in golden.corpus())
    for order in (3, 4):
        t = cc.build_ngram_table_from_corpus(corpus, order)
        txt = cc.format_ngram_file(t, nonzero_only=True)
        assert np.array_equal(cc.parse_ngram_file(txt, order).scores, t.scores)
        assert t.scores.sum() == len(corpus) - order + 1
    with pytest.raises(ValueError):
        cc.parse_ngram_file("abc 1\nab 2\n", 3)
    with pytest.raises(ValueError):
        cc.parse_ngram_file("abc -1\n", 3)
    with pytest.warns(UserWarning):
        cc.parse_ngram_file("abc 1\nabc 2\n", 3)


def test_packed_batches_and_ragged():
    flat, off = _lib.ragged([np.array([1, 2]), [3], np.zeros(0, np.int64)])
    assert flat.tolist() == [1, 2, 3] and off.tolist() == [0, 2, 3, 3]
    p = _lib.Packed.of([[0, 25], [7]])
    assert len(p) == 2 and p[0].tolist() == [0, 25] and p[1].tolist() == [7]
    assert _lib.ragged(p)[0] is p.flat
    for bad in ([[26]], [[-1]]):
        with pytest.raises(ValueError):
            _lib.ragged(bad)
    with pytest.raises(ValueError):
        _lib.Packed(np.array([1, 2], np.uint8), np.array([0, 3]))   # offsets past the end
    with pytest.raises(ValueError):
        _lib.Packed(np.array([1, 2], np.uint8), np.array([1, 2]))   # not starting at 0


def test_ngram_tables_validate():
    with pytest.raises(ValueError):
        cc.NgramTable(5, np.zeros(26**2, np.int64))
    with pytest.raises(ValueError):
        cc.NgramTable(3, np.zeros(26**2, np.int64))
    with pytest.raises(ValueError):
        cc.NgramTable(3, -np.ones(26**3, np.int64))
    with pytest.raises(ValueError):
        cc.LogNgramTable(3, np.ones(26**3), -24.0)          # positive log-probabilities
    t = cc.build_ngram_table_from_corpus("the theme then", 3)
    lg = cc.build_log_ngram_table(t, floor=-30.0)
    q = cc.quantize_log_table(lg)
    assert q.order == 3 and q.scores.max() <= 65535 and q.scores.min() >= 0
    # the affine map keeps the order of the log-probabilities (ties allowed by rounding)
    order = np.argsort(lg.logs, kind="stable")
    assert (np.diff(q.scores[order]) >= 0).all()
    with pytest.raises(ValueError):
        cc.build_log_ngram_table(t, floor=-1.0)                # floor above the rarest trigram
    assert cc.as_ngram_table(cc.BigramTable(np.arange(676))).order == 2


def test_batch_solver_validation_happens_before_the_gpu():
    logs = cc.LogBigramTable(np.full(676, -10.0), -24.0)
    cfg = cc.SctSolverConfig(key_length=5)
    with pytest.raises(ValueError):
        cc.solve_sct_batch([np.zeros(4, np.int64)], logs, cfg)               # shorter than the key
    with pytest.raises(ValueError):
        cc.solve_sct_batch([np.zeros(40, np.int64)] * 2, logs, cfg, seeds=[1])
    table = cc.BigramTable(np.ones(676, np.int64))
    with pytest.raises(ValueError):
        cc.solve_stochastic_batch([np.zeros(5, np.int64)], table, cc.MasSolverConfig())  # 1 letter
    assert cc.solve_stochastic_batch([], table, cc.MasSolverConfig()) == []
    with pytest.raises(ValueError):
        cc.encrypt_batch([[1, 2]], "xyz", key_seeds=[1])


def test_job_histories_are_lazy_lists():
    """engine.JobHistories (mas_det_solve's per-job histories, built on access) behaves as the
    list of [(iteration, score), ...] lists it replaces, across device parts."""
    it = np.array([0, 8, 9, 10], dtype=np.int32)
    sc = it.astype(np.int64) * 10
    off = np.array([0, 1, 1, 4], dtype=np.int64)
    h = engine.JobHistories([(it, sc, off), (it[:0], sc[:0], off[:1]), (it, sc, off)])
    want = [[(0, 0)], [], [(8, 80), (9, 90), (10, 100)]] * 2
    assert len(h) == 6 and list(h) == want and h == want
    assert h[-1] == want[-1] and h[1:3] == want[1:3]
    assert all(isinstance(v, int) for pair in h[2] for v in pair)
    with pytest.raises(IndexError):
        h[6]
    assert len(engine.JobHistories()) == 0


def test_scripts_and_bench_compile():
    """The measurement and evidence scripts (bench.py, scripts/*.py) at least compile, so a
    round-end run never dies on a syntax error."""
    import py_compile

    files = ([ROOT / "bench.py", ROOT / "__graft_entry__.py"] + sorted((ROOT / "scripts").glob("*.py"))
             + sorted((ROOT / "tests" / "tools").glob("*.py")))
    for f in files:
        py_compile.compile(str(f), doraise=True)


def _bench(*argv, env=None, timeout=300):
    import os
    import subprocess
    import sys

    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *argv], capture_output=True,
                          text=True, env=e, timeout=timeout)


def test_bench_gpus_n_fails_loudly_without_n_devices():
    """A plain `bench.py --gpus N` re-launches itself with N ranks, and refuses to run (exit 2,
    clear message) when fewer than N GPUs are visible -- it never silently measures one."""
    r = _bench("--gpus", "2", "--ciphers", "4", env={"CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2, r.stderr
    assert "--gpus 2 requested but only 0 CUDA device(s)" in r.stderr


def test_bench_reference_arm_covers_the_whole_batch():
    """--impl reference: the timed steps are disjoint slices that together cover every
    ciphertext, so its success curve is over the GPU arm's exact set; n_gpus is --gpus under
    either launcher, and under torchrun only rank 0 prints."""
    import json

    r = _bench("--impl", "reference", "--ciphers", "12", "--workers", "4", "--climbings", "500",
               "--steps", "5", "--warmup", "1")
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 1
    assert line["cpu_baseline"]["sample"].startswith("all 12 ciphertexts")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    # the same ciphertexts, workers and streams as the GPU arm: recovery from the oracle directly
    import bench

    plains, ciphers, scores, lengths = bench.make_workload(12)
    _, best = bench.cpu_port(ciphers, scores, 4, 500, range(12))
    rec = [np.array_equal(best[i][ciphers[i]], plains[i]) for i in range(12)]
    assert line["success_by_len"] == bench.success_curve(rec, lengths)
    r2 = _bench("--impl", "reference", "--gpus", "2", "--ciphers", "6", "--workers", "2",
                "--climbings", "200", "--steps", "2", "--warmup", "1")
    assert r2.returncode == 0, r2.stderr
    lines = [json.loads(x) for x in r2.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2


def test_quantize_sct_table_shift_and_range():
    import paper_2103_13937_b200 as cc

    lt = cc.LogBigramTable(-np.random.default_rng(3).random(676) * 20 - 1, -24.0)
    q = cc.quantize_sct_table(lt, text_len=400)
    assert q.order == 2 and q.shift == 16 and q.table.dtype == np.int32
    assert np.array_equal(q.table, np.rint(lt.logs * 2**16).astype(np.int32))
    assert 399 * int(np.abs(q.table).max()) < 2**31
    long = cc.quantize_sct_table(lt, text_len=60_000)
    assert long.shift < 16 and 59_999 * int(np.abs(long.table).max()) < 2**31


@pytest.mark.parametrize("order", [2, 3])
def test_fast_sct_oracle_reduces_to_reference_climb_on_dyadic_tables(order):
    """The fast mode's definition (cco_sct_fast_worker: quantised integer fitness) takes the
    reference climb's decisions exactly when the quantisation is exact and float64 sums are
    exact (log-probabilities that are multiples of 2^-10): keys equal, scores scaled by 2^10.
    The parity oracle itself is pinned to the reference by test_oracle_golden.py."""
    import paper_2103_13937_b200 as cc

    rng = np.random.default_rng(90 + order)
    logs = -rng.integers(1, 24 * 1024, 26**order) / 1024.0
    lt = cc.LogNgramTable(order, logs, -24.0) if order > 2 else cc.LogBigramTable(logs, -24.0)
    q = cc.quantize_sct_table(lt, text_len=600, max_shift=10)
    for k, n in [(5, 200), (10, 400), (17, 333)]:
        cipher = rng.integers(0, 26, n)
        fk, fs, fl = O.sct_fast_worker(cipher, q.table, order, k, 1500, 11, k)
        pk, ps, pl = O.sct_worker(cipher, logs, k, 1500, 11, k, order=order)
        assert np.array_equal(fk, pk) and fl == pl and fs == ps * 1024
        # the returned score is the integer fitness of the returned key
        plain = O.sct_decrypt(cipher, fk)
        assert fs == O.ngram_score_text(plain, order, q.table)


def test_restarts_with_stop_compute_nothing_past_the_stop():
    """mas._batched_restarts (solve_with_restarts / solve_sct): with `stop`, launches grow
    1, 2, 4, ... restarts, so at most the stopping restart's launch computes restarts past it
    (never reported); each elapsed is its launch's wall time (search.py:61-86)."""
    import time as _t

    from paper_2103_13937_b200.mas import _batched_restarts

    calls = []

    def make_batch(rs):
        calls.append(list(rs))
        _t.sleep(0.002 * len(rs))
        return [cc.SolveResult(np.array([r]), 10 - abs(r - 3), [10 - abs(r - 3)], []) for r in rs]

    best, runs = _batched_restarts(make_batch, 50, 64, stop=lambda res: res.best_score == 10)
    assert calls == [[0], [1, 2], [3, 4, 5, 6]] and len(runs) == 4 and best.restart_index == 3
    assert all(r.elapsed >= 0.0015 for r in runs) and runs[3].elapsed >= 0.007
    calls.clear()
    best, runs = _batched_restarts(make_batch, 50, 64, stop=None)
    assert len(runs) == 50 and len(calls) < 50 and best.restart_index == 3
    # the SCT solvers' constant launches (grow=False): one 64-worker restart per launch,
    # 64 workers' worth of smaller restarts
    calls.clear()
    best, runs = _batched_restarts(make_batch, 50, 64, stop=lambda res: res.best_score == 10,
                                   grow=False)
    assert calls == [[0], [1], [2], [3]] and len(runs) == 4 and best.restart_index == 3
    calls.clear()
    _batched_restarts(make_batch, 50, 16, stop=lambda res: res.best_score == 10, grow=False)
    assert calls == [[0, 1, 2, 3]]
