"""Restart sharding across processes: one process per GPU, torch.distributed for the plumbing.

The hot path has no data-path exchange: every worker is independent (rng.py:27-33 keys each
worker's stream by (seed, restart, worker)), so each rank climbs a contiguous slice of the
global worker index range on its own GPU.  The only collective is the final best-key
selection -- the reference's max_element (search.py:19-25, first maximum) lifted to a
lexicographic (max score, min global worker index) reduction over ranks -- plus an
all-gather of the per-worker scores the reference's SolveResult reports
(per_worker_scores, mas.py:273-278).  Payloads are a few bytes per worker, so this is
latency-bound; NCCL (or gloo on CPU) all_gather is used as is.

For one ciphertext, `solve_stochastic_sharded` / `solve_sct_sharded` return the same
SolveResult as mas.solve_stochastic / one restart of sct.solve_sct on one GPU, for any world
size.
"""
from __future__ import annotations

import numpy as np

from .engine import shard_bounds
from .rng import philox_keys, worker_stream_index
from .search import SolveResult


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def rank_world() -> tuple[int, int]:
    d = _dist()
    return (d.get_rank(), d.get_world_size()) if d else (0, 1)


def rank_slice(n_items: int, align: int = 1) -> tuple[int, int]:
    """This rank's contiguous [lo, hi) share of n_items (boundaries on `align`)."""
    rank, world = rank_world()
    bounds = shard_bounds(n_items, world, align)
    return bounds[rank] if rank < len(bounds) else (n_items, n_items)


def _device():
    import torch

    d = _dist()
    if d and d.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def all_gather_array(local: np.ndarray) -> np.ndarray:
    """Concatenate every rank's 1-d array in rank order (variable lengths allowed)."""
    d = _dist()
    if d is None:
        return local
    import torch

    dev = _device()
    world = d.get_world_size()
    n = torch.tensor([local.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    d.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes) if sizes else 0
    as_i64 = np.ascontiguousarray(local).view(np.int64) if local.dtype.itemsize == 8 else None
    if as_i64 is None:
        raise TypeError("all_gather_array expects 8-byte elements")
    buf = torch.zeros(m, dtype=torch.int64, device=dev)
    buf[: local.size] = torch.from_numpy(as_i64.copy()).to(dev)
    outs = [torch.zeros(m, dtype=torch.int64, device=dev) for _ in range(world)]
    d.all_gather(outs, buf)
    parts = [o[:s].cpu().numpy() for o, s in zip(outs, sizes)]
    return np.concatenate(parts).view(local.dtype) if parts else local[:0]


def best_over_ranks(score, index: int, payload: np.ndarray):
    """Lexicographic (max score, min global index) over ranks; returns the winner's
    (score, index, payload) on every rank.  Scores may be int or float."""
    d = _dist()
    if d is None:
        return score, index, payload
    import torch

    dev = _device()
    world = d.get_world_size()
    mine = torch.tensor([float(score), float(index)], dtype=torch.float64, device=dev)
    exact = torch.tensor([int(score)] if isinstance(score, (int, np.integer)) else [0],
                         dtype=torch.int64, device=dev)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    alle = [torch.zeros_like(exact) for _ in range(world)]
    d.all_gather(allv, mine)
    d.all_gather(alle, exact)
    is_int = isinstance(score, (int, np.integer))
    cand = []
    for r in range(world):
        s = int(alle[r].item()) if is_int else float(allv[r][0].item())
        cand.append((s, int(allv[r][1].item()), r))
    best = max(cand, key=lambda c: (c[0], -c[1]))
    owner = best[2]
    buf = torch.from_numpy(np.ascontiguousarray(payload, dtype=np.int64)).to(dev)
    d.broadcast(buf, src=owner)
    return best[0], best[1], buf.cpu().numpy()


def solve_stochastic_sharded(cipher, table, cfg, restart: int = 0, climb=None) -> SolveResult:
    """mas.solve_stochastic with the cfg.workers workers split over ranks.

    `climb` defaults to engine.mas_climb (this rank's GPU); tests substitute the oracle."""
    from . import engine
    from .mas import _check_cipher
    from .ngrams import as_ngram_table

    climb = climb or engine.mas_climb
    text = _check_cipher(cipher)
    t = as_ngram_table(table)
    W = cfg.workers
    lo, hi = rank_slice(W)
    streams = [worker_stream_index(restart, w) for w in range(lo, hi)]
    if hi > lo:
        extra = {} if t.order == 2 else {"order": t.order}
        res = climb([text], np.zeros(hi - lo, np.int32), philox_keys([cfg.global_seed], streams),
                    t.scores, cfg.climbings, group_size=hi - lo, **extra)
        local_scores = np.asarray(res.scores, dtype=np.int64)
        b = int(res.group_best[0])
        best_local = (int(local_scores[b]), lo + b, np.asarray(res.keys[b], dtype=np.int64))
    else:
        local_scores = np.zeros(0, dtype=np.int64)
        best_local = (np.iinfo(np.int64).min, np.iinfo(np.int64).max, np.zeros(26, np.int64))
    per_worker = all_gather_array(local_scores)
    score, idx, mapping = best_over_ranks(best_local[0], best_local[1], best_local[2])
    return SolveResult(best_text=mapping[text], best_score=int(score),
                       per_worker_scores=[int(v) for v in per_worker], history=[])


def solve_sct_sharded(cipher, logs, cfg, restart: int = 0, climb=None) -> SolveResult:
    """One restart of sct.solve_sct (sct.py:179-210) with the cfg.workers workers split over
    ranks: per-worker float64 scores gathered in worker order, best key = first maximum.

    `climb` defaults to engine.sct_climb (this rank's GPU); tests substitute the oracle."""
    from . import engine
    from .ciphers import sct_decrypt
    from .ngrams import as_log_ngram_table

    climb = climb or engine.sct_climb
    text = np.asarray(cipher, dtype=np.int64)
    if text.size < cfg.key_length:
        raise ValueError("ciphertext shorter than the key")
    lt = as_log_ngram_table(logs)
    W, k = cfg.workers, cfg.key_length
    lo, hi = rank_slice(W)
    streams = [worker_stream_index(restart, w) for w in range(lo, hi)]
    if hi > lo:
        res = climb([text], np.zeros(hi - lo, np.int32), philox_keys([cfg.global_seed], streams),
                    lt.logs, k, cfg.climbings, p1=cfg.p1, p2=cfg.p2, op1_hop=cfg.op1_hop,
                    op2_hop=cfg.op2_hop, group_size=hi - lo, order=lt.order)
        local_scores = np.asarray(res.scores, dtype=np.float64)
        b = int(res.group_best[0])
        best_local = (float(local_scores[b]), lo + b, np.asarray(res.keys[b], dtype=np.int64)[:k])
    else:
        local_scores = np.zeros(0, dtype=np.float64)
        best_local = (-np.inf, np.iinfo(np.int64).max, np.zeros(k, np.int64))
    per_worker = all_gather_array(local_scores)
    score, idx, key = best_over_ranks(best_local[0], best_local[1], best_local[2])
    return SolveResult(best_text=sct_decrypt(text, key), best_score=float(score),
                       per_worker_scores=[float(v) for v in per_worker], history=[],
                       best_key=key)
