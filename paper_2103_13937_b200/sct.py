"""Single-columnar-transposition attack (reference sct.py:1-210), GPU-backed.

sct_worker / solve_sct run on the GPU: decryption by index arithmetic, float64 scoring in
numpy's pairwise order, one warp per worker (csrc/ccg_sct.cu) or one worker per lane for
large batches (csrc/ccg_sct_lane.cu).  The operator functions below are the reference's
host-side helpers, drawing from a (GPU-generated) WorkerRng stream; the climb itself never
calls them.  solve_sct_fast is the opt-in fast mode (quantised fitness, incremental
rescoring; not bit-exact with the reference by design).

n-gram extension: sct_worker / solve_sct also accept an ngrams.LogNgramTable of order 3 or
4 (BASELINE.json config 3: trigram scoring); the candidate score is then the pairwise sum of
the window log-probabilities of that order.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import engine
from .ciphers import sct_decrypt
from .codec import MappedText
from .ngrams import LogBigramTable, as_log_ngram_table, quantize_sct_table
from .rng import WorkerRng, philox_keys, worker_stream_index
from .search import RestartSummary, SolveResult
from .mas import _batched_restarts


class Operator(enum.Enum):
    ELEMENT_SWAP = 1
    BLOCK_SWAP = 2
    BLOCK_SHIFT = 3


@dataclass
class SctSolverConfig:
    """sct.py:43-66."""

    key_length: int
    workers: int = 64
    climbings: int = 15_000
    p1: int = 33
    p2: int = 66
    op1_hop: int = 3
    op2_hop: int = 3
    restarts: int = 1
    global_seed: int = 0

    def __post_init__(self):
        if self.key_length < 2:
            raise ValueError("key_length must be at least 2")
        if not 0 <= self.p1 <= self.p2 <= 100:
            raise ValueError("thresholds must satisfy 0 <= p1 <= p2 <= 100")
        if self.climbings < 0:
            raise ValueError("climbings must be non-negative")
        for name in ("workers", "op1_hop", "op2_hop", "restarts"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be at least 1")


def select_operator(u_percent: int, p1: int, p2: int) -> Operator:
    """[0,p1) -> I, [p1,p2) -> II, [p2,100) -> III (sct.py:69-79)."""
    if not 0 <= p1 <= p2 <= 100:
        raise ValueError("thresholds must satisfy 0 <= p1 <= p2 <= 100")
    if not 0 <= u_percent < 100:
        raise ValueError("u_percent must lie in [0, 100)")
    if u_percent < p1:
        return Operator.ELEMENT_SWAP
    return Operator.BLOCK_SWAP if u_percent < p2 else Operator.BLOCK_SHIFT


def apply_element_swaps(key: np.ndarray, state: WorkerRng, max_hops: int) -> np.ndarray:
    """1..max_hops random position swaps (sct.py:82-89)."""
    out = np.array(key, dtype=np.int64, copy=True)
    for _ in range(1 + state.next_int_below(max_hops)):
        i, j = state.next_distinct_pair(out.size)
        out[[i, j]] = out[[j, i]]
    return out


def apply_block_swaps(key: np.ndarray, state: WorkerRng, max_hops: int) -> np.ndarray:
    """1..max_hops swaps of equal, non-overlapping blocks (sct.py:92-112)."""
    out = np.array(key, dtype=np.int64, copy=True)
    k = out.size
    for _ in range(1 + state.next_int_below(max_hops)):
        length = 1 + state.next_int_below(k // 2)
        while True:
            p, q = state.next_distinct_pair(k - length + 1)
            if abs(p - q) >= length:
                break
        p, q = min(p, q), max(p, q)
        out[p:p + length], out[q:q + length] = out[q:q + length].copy(), out[p:p + length].copy()
    return out


def apply_block_shift(key: np.ndarray, state: WorkerRng) -> np.ndarray:
    """Move one block to a different in-bounds position (sct.py:115-135)."""
    out = np.array(key, dtype=np.int64, copy=True)
    k = out.size
    length = 1 + state.next_int_below(k - 1)
    starts = k - length + 1
    p = state.next_int_below(starts)
    dest = state.next_int_below(starts)
    while dest == p:
        dest = state.next_int_below(starts)
    lo, hi = min(p, dest), max(p, dest) + length
    out[lo:hi] = np.roll(out[lo:hi], -length if dest > p else length)
    return out


def sct_worker(cipher: MappedText, logs: LogBigramTable, cfg: SctSolverConfig,
               state: WorkerRng) -> tuple[np.ndarray, float]:
    """One worker's climb from permutation(k) (sct.py:148-170) as a one-warp GPU launch;
    `state` is advanced by exactly the draws consumed."""
    text = np.asarray(cipher, dtype=np.int64)
    if text.size < cfg.key_length:
        raise ValueError("ciphertext shorter than the key")
    lt = as_log_ngram_table(logs)
    res = engine.sct_climb([text], [0], [state.key], lt.logs, cfg.key_length, cfg.climbings,
                           p1=cfg.p1, p2=cfg.p2, op1_hop=cfg.op1_hop, op2_hop=cfg.op2_hop,
                           skips=[state.position], draws_used=True, order=lt.order)
    state.advance(int(res.draws_used[0]))
    return res.keys[0].astype(np.int64), float(res.scores[0])


def _restart_batch(text, logs, cfg, restarts):
    W = cfg.workers
    streams = [worker_stream_index(r, w) for r in restarts for w in range(W)]
    keys = philox_keys([cfg.global_seed], streams)
    lt = as_log_ngram_table(logs)
    res = engine.sct_climb([text], np.zeros(len(streams), np.int32), keys, lt.logs,
                           cfg.key_length, cfg.climbings, p1=cfg.p1, p2=cfg.p2,
                           op1_hop=cfg.op1_hop, op2_hop=cfg.op2_hop, group_size=W, order=lt.order)
    out = []
    for i, _ in enumerate(restarts):
        sc = res.scores[i * W:(i + 1) * W]
        best = int(res.group_best[i])
        key = res.keys[i * W + best].astype(np.int64)
        out.append(SolveResult(
            best_text=sct_decrypt(text, key),
            best_score=float(sc[best]),
            per_worker_scores=[float(v) for v in sc],
            history=[],
            best_key=key,
        ))
    return out


def solve_sct(cipher: MappedText, logs: LogBigramTable, cfg: SctSolverConfig, jobs: int = 1,
              stop=None) -> tuple[SolveResult, list[RestartSummary]]:
    """Workers x restarts on the GPU; lowest worker index wins ties, earliest restart wins
    ties, `stop` applied restart by restart (sct.py:179-210)."""
    text = np.asarray(cipher, dtype=np.int64)
    if text.size < cfg.key_length:
        raise ValueError("ciphertext shorter than the key")
    return _batched_restarts(lambda rs: _restart_batch(text, logs, cfg, rs), cfg.restarts,
                             cfg.workers, stop, grow=False)


def solve_sct_batch(ciphers, logs, cfg: SctSolverConfig, restart: int = 0, seeds=None,
                    key_lengths=None) -> list[SolveResult]:
    """One restart of solve_sct (sct.py:179-210) for many ciphertexts (any mix of lengths) in
    one GPU launch; key_lengths (default cfg.key_length) may differ per ciphertext.
    Ciphertext i uses the streams (restart << 32) | w of seed `seeds[i]` (default
    cfg.global_seed)."""
    texts = [np.asarray(c, dtype=np.int64) for c in ciphers]
    n, W = len(texts), cfg.workers
    if n == 0:
        return []
    seeds = [cfg.global_seed] * n if seeds is None else list(seeds)
    klens = [cfg.key_length] * n if key_lengths is None else [int(k) for k in key_lengths]
    if len(seeds) != n or len(klens) != n:
        raise ValueError("one seed and key length per ciphertext required")
    for t, k in zip(texts, klens):
        if k < 2:
            raise ValueError("key_length must be at least 2")
        if t.size < k:
            raise ValueError("ciphertext shorter than the key")
    streams = [worker_stream_index(restart, w) for w in range(W)]
    keys = np.concatenate([philox_keys([s], streams) for s in seeds])
    lt = as_log_ngram_table(logs)
    res = engine.sct_climb(texts, np.repeat(np.arange(n, dtype=np.int32), W), keys, lt.logs,
                           np.repeat(np.array(klens, dtype=np.int32), W), cfg.climbings,
                           p1=cfg.p1, p2=cfg.p2, op1_hop=cfg.op1_hop, op2_hop=cfg.op2_hop,
                           group_size=W, order=lt.order)
    out = []
    for i, text in enumerate(texts):
        sc = res.scores[i * W:(i + 1) * W]
        best = int(res.group_best[i])
        key = res.keys[i * W + best, :klens[i]].astype(np.int64)
        out.append(SolveResult(best_text=sct_decrypt(text, key), best_score=float(sc[best]),
                               per_worker_scores=[float(v) for v in sc], history=[],
                               best_key=key))
    return out


def solve_sct_fast(cipher: MappedText, logs: LogBigramTable, cfg: SctSolverConfig, jobs: int = 1,
                   stop=None, shift: int | None = None) -> tuple[SolveResult, list[RestartSummary]]:
    """solve_sct (sct.py:179-210) in the opt-in fast mode: the same workers, streams,
    operators and restart rules, with the fitness replaced by the int32-quantised log table
    (ngrams.quantize_sct_table; `shift` defaults to the largest safe one) and candidates
    scored incrementally on the GPU (engine.sct_fast_climb).  Scores are
    reported as quantised sums / 2^shift (log2 units); decisions can differ from the
    reference's float64 climb where two candidates' scores are within the rounding."""
    text = np.asarray(cipher, dtype=np.int64)
    if text.size < cfg.key_length:
        raise ValueError("ciphertext shorter than the key")
    lt = as_log_ngram_table(logs)
    q = quantize_sct_table(lt, text_len=max(text.size, lt.order), **(
        {} if shift is None else {"max_shift": int(shift)}))
    scale = 2.0 ** -q.shift
    W = cfg.workers

    def batch(restarts):
        streams = [worker_stream_index(r, w) for r in restarts for w in range(W)]
        res = engine.sct_fast_climb([text], np.zeros(len(streams), np.int32),
                                    philox_keys([cfg.global_seed], streams), q, cfg.key_length,
                                    cfg.climbings, p1=cfg.p1, p2=cfg.p2, op1_hop=cfg.op1_hop,
                                    op2_hop=cfg.op2_hop, group_size=W, lookups=False)
        out = []
        for i, _ in enumerate(restarts):
            sc = res.scores[i * W:(i + 1) * W]
            best = int(res.group_best[i])
            key = res.keys[i * W + best].astype(np.int64)
            out.append(SolveResult(best_text=sct_decrypt(text, key), best_score=float(sc[best]) * scale,
                                   per_worker_scores=[float(v) * scale for v in sc], history=[],
                                   best_key=key))
        return out

    return _batched_restarts(batch, cfg.restarts, W, stop, grow=False)
