"""Monoalphabetic-substitution attack (reference mas.py:1-299), GPU-backed.

Stochastic better-neighbour climbing (mas.py:218-299) runs entirely on the GPU: one
warp per worker (csrc/ccg_mas_tform.cu, csrc/ccg_mas.cu).  The deterministic best-neighbour
variant (mas.py:84-169) runs one CTA of 325 pair-workers per restart with the whole
iteration loop on the device (csrc/ccg_mas_det.cu).  Signatures, defaults, validation messages and
result objects follow the reference so this module drops in for it; `jobs` is accepted
for signature compatibility and has no effect on results (the reference guarantees the
same: search.py:4-7).

n-gram extension: every stochastic entry point also accepts an ngrams.NgramTable of order
3 or 4 (BASELINE.json configs 4-5; the reference has bigrams only); the climb
then runs the position-based n-gram kernel (csrc/ccg_mas_ngram.cu) with the same proposal
stream and accept rule.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import engine
from .codec import ALPHABET_SIZE, MappedText
from .ngrams import BigramTable, as_ngram_table
from .pairs import PAIR_TOTAL, index_to_pair
from .rng import WorkerRng, philox_keys, pivot_stream_index, worker_stream_index
from .search import RestartSummary, SolveResult, fold_restarts


@dataclass
class MasSolverConfig:
    """mas.py:39-65."""

    mode: str = "stochastic"
    workers: int = 64
    iterations: int = 500
    climbings: int = 10_000
    restarts: int = 1
    global_seed: int = 0

    def __post_init__(self):
        if self.mode not in ("deterministic", "stochastic"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.mode == "deterministic" and self.workers != PAIR_TOTAL:
            raise ValueError(
                f"deterministic mode requires workers={PAIR_TOTAL} (one per letter pair)"
            )
        for name in ("workers", "iterations", "climbings", "restarts"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be at least 1")


def _check_cipher(cipher) -> np.ndarray:
    text = np.asarray(cipher, dtype=np.int64)
    if text.size < 2 or np.unique(text).size < 2:
        raise ValueError("ciphertext must contain at least two distinct letters")
    return text


def bigram_count_matrix(text: MappedText) -> np.ndarray:
    """26x26 adjacent-pair counts (mas.py:172-178)."""
    t = np.asarray(text, dtype=np.int64)
    if t.size < 2:
        return np.zeros((ALPHABET_SIZE, ALPHABET_SIZE), dtype=np.int64)
    flat = np.bincount(t[:-1] * ALPHABET_SIZE + t[1:], minlength=ALPHABET_SIZE * ALPHABET_SIZE)
    return flat.astype(np.int64).reshape(ALPHABET_SIZE, ALPHABET_SIZE)


def swap_delta(counts: np.ndarray, a: int, b: int, score_matrix: np.ndarray) -> int:
    """Exact score change of interchanging letters a, b (mas.py:181-210), on the GPU."""
    return int(engine.mas_delta_counts_batch(counts, [(a, b)], score_matrix)[0])


def text_swap_delta(text: MappedText, a: int, b: int, table: BigramTable) -> int:
    """swap_delta on the text's own count matrix (mas.py:315-317), on the GPU."""
    return int(engine.mas_delta_batch([text], [(a, b)], table.scores)[0])


def stochastic_worker(cipher: MappedText, table: BigramTable, climbings: int,
                      state: WorkerRng) -> tuple[np.ndarray, int]:
    """One worker's climb from the ciphertext (mas.py:218-244) as a one-warp GPU launch.
    `state` is advanced by exactly the draws the worker consumed."""
    text = np.asarray(cipher, dtype=np.int64)
    t = as_ngram_table(table)
    res = engine.mas_climb([text], [0], [state.key], t.scores, climbings, order=t.order,
                           skips=[state.position], draws_used=True)
    state.advance(int(res.draws_used[0]))
    return res.keys[0].astype(np.int64)[text], int(res.scores[0])


def _restart_batch(text, table, cfg, restarts, early_exit=True):
    """All workers of the given restarts in one engine call; one SolveResult each."""
    W = cfg.workers
    streams = [worker_stream_index(r, w) for r in restarts for w in range(W)]
    keys = philox_keys([cfg.global_seed], streams)
    t = as_ngram_table(table)
    res = engine.mas_climb([text], np.zeros(len(streams), np.int32), keys, t.scores,
                           cfg.climbings, order=t.order, group_size=W, early_exit=early_exit)
    out = []
    for i, _ in enumerate(restarts):
        sc = res.scores[i * W:(i + 1) * W]
        best = int(res.group_best[i])
        out.append(SolveResult(
            best_text=res.keys[i * W + best].astype(np.int64)[text],
            best_score=int(sc[best]),
            per_worker_scores=[int(v) for v in sc],
            history=[],
        ))
    return out


def solve_stochastic(cipher: MappedText, table: BigramTable, cfg: MasSolverConfig, jobs: int = 1,
                     restart: int = 0) -> SolveResult:
    """cfg.workers independent climbs with streams (restart << 32) | w; the first maximum
    wins (mas.py:253-278)."""
    text = _check_cipher(cipher)
    return _restart_batch(text, table, cfg, [restart])[0]


def _batched_restarts(make_batch, restarts: int, workers: int, stop, grow: bool = True):
    """Evaluate restarts in launches of several restarts and fold them in order
    (search.py:61-86).  Results equal the sequential reference: restarts are independent of
    each other and of `stop`, which is applied restart by restart in order.

    With a `stop` callback the first launch is a single restart (a solve usually stops after
    it) and, with `grow`, the launches grow 1, 2, 4, ... restarts; at most one launch ever
    computes restarts past the stopping one (they are discarded, never reported).  The SCT
    solvers pass grow=False: their latency kernels give a restart of 64 workers a pair of SMs
    each, so two restarts in one launch take about as long as two launches of one, and four
    fall back to slower kernels.  Without `stop` every launch is about one full wave.
    RestartSummary.elapsed is the wall time of the launch that computed the restart (its
    restarts ran concurrently for that long), the analogue of the reference's per-restart
    timing (search.py:75-78)."""
    target = 8192 * max(1, len(engine.devices()))  # workers per chunk: ~one full wave
    chunk = max(1, min(restarts, target // max(1, workers)))
    first = 1 if grow else max(1, min(chunk, 64 // max(1, workers)))

    def gen():
        r = 0
        size = first if stop is not None else chunk
        while r < restarts:
            rs = list(range(r, min(restarts, r + size)))
            if grow:
                size = min(chunk, 2 * size)
            t0 = time.perf_counter()
            results = make_batch(rs)
            dt = time.perf_counter() - t0
            for res in results:
                yield res, dt
            r += len(rs)

    return fold_restarts(gen(), stop)


def solve_with_restarts(cipher: MappedText, table: BigramTable, cfg: MasSolverConfig,
                        jobs: int = 1, stop=None) -> tuple[SolveResult, list[RestartSummary]]:
    """mas.py:281-299."""
    text = _check_cipher(cipher)
    if cfg.mode == "deterministic":
        return _batched_restarts(lambda rs: _det_batch(text, table, cfg, rs), cfg.restarts,
                                 PAIR_TOTAL, stop)
    return _batched_restarts(lambda rs: _restart_batch(text, table, cfg, rs), cfg.restarts,
                             cfg.workers, stop)


# ------------------------------------------------------------------ deterministic mode
def deterministic_step(current: MappedText, pivot: tuple[int, int],
                       table: BigramTable) -> tuple[np.ndarray, int, int]:
    """Evaluate all 325 pair-workers for one pivot on the GPU; return the first best
    (candidate text, score, worker index) (mas.py:84-120)."""
    text = np.asarray(current, dtype=np.int64)
    pl, pr = int(pivot[0]), int(pivot[1])
    if pl == pr:
        raise ValueError("pivot letters must differ")
    present = np.zeros(ALPHABET_SIZE, dtype=bool)
    present[text] = True
    if not (0 <= pl < ALPHABET_SIZE and 0 <= pr < ALPHABET_SIZE and present[pl] and present[pr]):
        raise ValueError("both pivot letters must occur in the text")
    scores = engine.mas_det_step_batch([text], [(pl, pr)], table.scores)[0]
    best_index = int(np.argmax(scores))  # first maximum (search.py:19-25)
    return climb_unchecked(text, best_index, (pl, pr)), int(scores[best_index]), best_index


def climb_unchecked(current, best_index, pivot):
    other_left, other_right = index_to_pair(best_index)
    pl, pr = int(pivot[0]), int(pivot[1])
    first = np.arange(ALPHABET_SIZE, dtype=np.int64)
    first[pl], first[other_left] = other_left, pl
    second = np.arange(ALPHABET_SIZE, dtype=np.int64)
    second[pr], second[other_right] = other_right, pr
    return second[first][np.asarray(current, dtype=np.int64)]


def climb(current: MappedText, best_index: int, pivot: tuple[int, int]) -> np.ndarray:
    """Reconstruct the winning worker's candidate from its index (mas.py:123-130)."""
    other_left, other_right = index_to_pair(best_index)
    pl, pr = int(pivot[0]), int(pivot[1])
    if pl == other_right or pr == other_left:
        raise ValueError(f"worker {best_index} is excluded for pivot ({pl}, {pr})")
    return climb_unchecked(current, best_index, pivot)


def _det_batch(text, table, cfg, restarts):
    keys = philox_keys([cfg.global_seed], [pivot_stream_index(r) for r in restarts])
    res = engine.mas_det_solve([text], np.zeros(len(restarts), np.int32), keys, table.scores,
                               cfg.iterations)
    return [SolveResult(best_text=res.maps[i].astype(np.int64)[text], best_score=int(res.scores[i]),
                        per_worker_scores=[], history=[(int(a), int(b)) for a, b in res.history[i]])
            for i in range(len(restarts))]


def solve_deterministic(cipher: MappedText, table: BigramTable, cfg: MasSolverConfig,
                        restart: int = 0) -> SolveResult:
    """The best-neighbour climb for cfg.iterations iterations (mas.py:140-169), the whole
    loop in one GPU launch (one CTA, 325 pair-workers)."""
    text = _check_cipher(cipher)
    return _det_batch(text, table, cfg, [restart])[0]


# ------------------------------------------------------------------ many ciphertexts
def solve_stochastic_batch(ciphers, table, cfg: MasSolverConfig, restart: int = 0,
                           seeds=None) -> list[SolveResult]:
    """solve_stochastic (mas.py:253-278) for many ciphertexts in one GPU launch: ciphertext i
    gets cfg.workers workers on the streams (restart << 32) | w of seed `seeds[i]` (default
    cfg.global_seed for all), exactly as separate solve_stochastic calls would.  The batch
    form of BASELINE.json configs 2 and 4."""
    texts = [_check_cipher(c) for c in ciphers]
    n, W = len(texts), cfg.workers
    if n == 0:
        return []
    seeds = [cfg.global_seed] * n if seeds is None else list(seeds)
    if len(seeds) != n:
        raise ValueError("one seed per ciphertext required")
    streams = [worker_stream_index(restart, w) for w in range(W)]
    keys = np.concatenate([philox_keys([s], streams) for s in seeds])
    t = as_ngram_table(table)
    res = engine.mas_climb(texts, np.repeat(np.arange(n, dtype=np.int32), W), keys, t.scores,
                           cfg.climbings, order=t.order, group_size=W, early_exit=True)
    out = []
    for i, text in enumerate(texts):
        sc = res.scores[i * W:(i + 1) * W]
        best = int(res.group_best[i])
        out.append(SolveResult(best_text=res.keys[i * W + best].astype(np.int64)[text],
                               best_score=int(sc[best]), per_worker_scores=[int(v) for v in sc],
                               history=[]))
    return out
