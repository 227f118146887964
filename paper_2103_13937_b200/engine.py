"""Batch entry points of the GPU engine and the in-process multi-GPU restart sharder.

A "worker" is one (ciphertext, Philox stream) hill climb, exactly one task of the
reference's run_worker_pool (search.py:49-58; mas.py:266-270, sct.py:194-198).  A batch of
workers is split into contiguous, group-aligned ranges, one per device, and each range is
one ccg_*_climb call on that device (one kernel launch + one group-argmax launch).  Host
threads drive the devices concurrently (ctypes releases the GIL).  Every worker's output
depends only on its own (ciphertext, key, stream), so results are identical for any
device count or split -- the property the reference tests as jobs=1 == jobs=2
(tests/test_mas.py:240-249, tests/test_sct.py:160-169).

Device selection: set_devices([...]) or the CCG_DEVICES environment variable
("0,1,2,3"); default is LOCAL_RANK (one process per GPU under torchrun) or device 0.
"""
from __future__ import annotations

import bisect
import collections.abc
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib

_devices: list[int] | None = None


def set_devices(devices) -> None:
    """Use these CUDA devices for subsequent batches (None = back to the default)."""
    global _devices
    _devices = None if devices is None else [int(d) for d in devices]


def devices() -> list[int]:
    if _devices is not None:
        return list(_devices)
    env = os.environ.get("CCG_DEVICES")
    if env:
        return [int(x) for x in env.split(",") if x.strip()]
    return [int(os.environ.get("LOCAL_RANK", "0"))]


def default_device() -> int:
    return devices()[0]


def shard_bounds(n_items: int, n_shards: int, align: int = 1) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) ranges over n_items, boundaries on multiples of `align`,
    as even as possible; empty ranges are dropped."""
    align = max(1, int(align))
    units = (n_items + align - 1) // align
    n_shards = max(1, min(int(n_shards), units)) if units else 1
    base, extra = divmod(units, n_shards)
    out, u = [], 0
    for s in range(n_shards):
        cnt = base + (1 if s < extra else 0)
        lo, hi = u * align, min(n_items, (u + cnt) * align)
        if hi > lo:
            out.append((lo, hi))
        u += cnt
    return out


@dataclass
class ClimbResult:
    scores: np.ndarray          # int64 (MAS) or float64 (SCT), per worker
    keys: np.ndarray            # uint8[n, 26] letter maps (MAS) / uint8[n, k] column keys (SCT)
    group_best: np.ndarray | None
    draws_used: np.ndarray | None
    last_accept: np.ndarray | None
    tries_done: np.ndarray | None
    launches: int
    accepts: np.ndarray | None = None   # accepted interchanges per worker (bigram MAS kernels)
    computed: np.ndarray | None = None  # n-gram kernel: deltas computed by position walks
    lookups: np.ndarray | None = None   # fast SCT: table lookups of the incremental rescoring


def _run_sharded(n_workers, group_size, devs, fn):
    bounds = shard_bounds(n_workers, len(devs), group_size if group_size > 0 else 1)
    if len(bounds) <= 1:
        return [fn(devs[0], 0, n_workers)]
    with ThreadPoolExecutor(max_workers=len(bounds)) as pool:
        futs = [pool.submit(fn, devs[i], lo, hi) for i, (lo, hi) in enumerate(bounds)]
        return [f.result() for f in futs]


def _concat(parts, name):
    vals = [getattr(p, name) for p in parts]
    if any(v is None for v in vals):
        return None
    return np.concatenate(vals)


def mas_climb(ciphers, cipher_of, keys, table_scores, climbings, *, skips=None, group_size=0,
              draws_used=False, last_accept=False, tries_done=False, early_exit=False,
              order=2, ngram_kernel=False, kernel="auto", accepts=False, computed=False,
              lookups=False, out: ClimbResult | None = None, devices_=None) -> ClimbResult:
    """Run stochastic_worker (mas.py:218-244) for every worker on the GPU(s).

    ciphers: list of letter arrays; cipher_of: int per worker; keys: uint64[n, 2] Philox
    keys (rng.philox_keys); table_scores: int64[26**order].  order 2 runs the bigram kernels
    (ccg_mas_climb); order 3/4 -- or ngram_kernel=True at order 2 -- the position-based
    n-gram kernel (ccg_mas_ngram_climb, entries must fit uint16).  `kernel` selects the
    bigram kernel ("auto", "dform", "dtable", "tform", "packed"); results are identical.
    `ciphers` may be a list of letter arrays or a pre-packed _lib.Packed batch; `out` may
    supply the result arrays (e.g. in pinned host memory) for the whole batch."""
    flat, off = _lib.ragged(ciphers)
    cof = np.ascontiguousarray(cipher_of, dtype=np.int32).reshape(-1)
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, 2)
    order = int(order)
    use_ng = ngram_kernel or order != 2
    table = np.ascontiguousarray(table_scores, dtype=np.int64).reshape(-1)
    if table.size != 26**order:
        raise ValueError(f"expected {26**order} table entries for order {order}, got {table.size}")
    if use_ng:
        if table.size and (table.min() < 0 or table.max() > 65535):
            raise _lib.EngineError("the n-gram kernel takes table entries in 0..65535 "
                                   "(quantise the table with ngrams.quantize_log_table)")
        table = np.ascontiguousarray(table, dtype=np.uint16)
    n = cof.size
    if keys.shape[0] != n:
        raise ValueError("one Philox key per worker required")
    sk = None if skips is None else np.ascontiguousarray(skips, dtype=np.uint64).reshape(-1)
    devs = devices_ or devices()

    given = out

    def view(arr, lo_, hi_):
        return None if arr is None else arr[lo_:hi_]

    def run(dev, lo, hi):
        m = hi - lo
        if given is not None:
            g0, g1 = (lo // group_size, hi // group_size) if group_size > 0 else (0, 0)
            out = ClimbResult(
                scores=given.scores[lo:hi], keys=given.keys[lo:hi],
                group_best=view(given.group_best, g0, g1) if group_size > 0 else None,
                draws_used=view(given.draws_used, lo, hi), last_accept=view(given.last_accept, lo, hi),
                tries_done=view(given.tries_done, lo, hi), launches=0,
                accepts=view(given.accepts, lo, hi) if not use_ng else None)
        else:
            out = ClimbResult(
                scores=np.empty(m, dtype=np.int64),
                keys=np.empty((m, 26), dtype=np.uint8),
                group_best=np.empty(m // group_size, dtype=np.int64) if group_size > 0 else None,
                draws_used=np.empty(m, dtype=np.uint64) if draws_used else None,
                last_accept=np.empty(m, dtype=np.int64) if last_accept else None,
                tries_done=np.empty(m, dtype=np.int64) if tries_done else None,
                launches=0,
                accepts=np.empty(m, dtype=np.int64) if (accepts and not use_ng) else None,
                computed=np.empty(m, dtype=np.int64) if (computed and use_ng) else None,
                lookups=np.empty(m, dtype=np.int64) if (lookups and use_ng) else None,
            )
        if m == 0:
            return out
        c_of = np.ascontiguousarray(cof[lo:hi])
        k = np.ascontiguousarray(keys[lo:hi])
        s = None if sk is None else np.ascontiguousarray(sk[lo:hi])
        a = _lib.MasNgramArgs() if use_ng else _lib.MasClimbArgs()
        if not use_ng:
            a.accepts = _lib.ptr(out.accepts)
        a.ciphers, a.offsets, a.n_ciphers = _lib.ptr(flat), _lib.ptr(off), off.size - 1
        a.cipher_of, a.keys, a.skips = _lib.ptr(c_of), _lib.ptr(k), _lib.ptr(s)
        a.n_workers, a.climbings, a.table = m, int(climbings), _lib.ptr(table)
        a.scores, a.maps = _lib.ptr(out.scores), _lib.ptr(out.keys)
        a.draws_used, a.last_accept = _lib.ptr(out.draws_used), _lib.ptr(out.last_accept)
        a.tries_done = _lib.ptr(out.tries_done)
        a.group_size, a.group_best = int(group_size), _lib.ptr(out.group_best)
        a.flags = (_lib.FLAG_EARLY_EXIT if early_exit else 0) | _lib.KERNEL_FLAGS[kernel]
        if use_ng:
            a.order = order
            a.computed = _lib.ptr(out.computed)
            a.lookups = _lib.ptr(out.lookups)
        ctx = _lib.context(dev)
        with ctx.lock:
            before = ctx.launches()
            fn = _lib.load().ccg_mas_ngram_climb if use_ng else _lib.load().ccg_mas_climb
            _lib.check(fn(ctx.handle, a), "mas_climb")
            out.launches = ctx.launches() - before
        return out

    parts = _run_sharded(n, group_size, devs, run)
    if given is not None:
        given.launches = sum(p.launches for p in parts)
        return given
    return ClimbResult(
        scores=_concat(parts, "scores"), keys=_concat(parts, "keys"),
        group_best=_concat(parts, "group_best"), draws_used=_concat(parts, "draws_used"),
        last_accept=_concat(parts, "last_accept"), tries_done=_concat(parts, "tries_done"),
        launches=sum(p.launches for p in parts), accepts=_concat(parts, "accepts"),
        computed=_concat(parts, "computed"), lookups=_concat(parts, "lookups"),
    )


def sct_climb(ciphers, cipher_of, keys, logs, key_length, climbings, *, p1=33, p2=66, op1_hop=3,
              op2_hop=3, skips=None, group_size=0, draws_used=False, last_accept=False,
              tries_done=False, order=2, speculate=True, kernel="auto", table_l2=False,
              devices_=None) -> ClimbResult:
    """Run sct_worker (sct.py:148-170) for every worker on the GPU(s).  logs:
    float64[26**order] (order 2 = the reference's bigram table).  key_length may be an int or
    one length per worker (a ragged batch in one launch); keys come back as
    uint8[n, max key length], row i valid in its first key_length[i] entries.  Ciphertexts
    may have any mix of lengths.  Kernels (identical results): with at most a few workers per
    SM and one common text length, each worker gets a CTA of warps that evaluate consecutive
    proposals speculatively from its proposal chain parsed ahead (speculate="replay": the
    kernel whose warps replay their predecessors' draws instead; speculate=False turns
    speculation off); otherwise one worker per lane
    (kernel="lane"); kernel="warp" forces the one-warp-per-worker kernel (one text length)."""
    flat, off = _lib.ragged(ciphers)
    cof = np.ascontiguousarray(cipher_of, dtype=np.int32).reshape(-1)
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, 2)
    lg = np.ascontiguousarray(logs, dtype=np.float64).reshape(-1)
    if lg.size != 26**int(order):
        raise ValueError(f"expected {26**int(order)} log-table entries for order {order}")
    n = cof.size
    klens = None
    if np.ndim(key_length):
        klens = np.ascontiguousarray(key_length, dtype=np.int32).reshape(-1)
        if klens.size != n:
            raise ValueError("one key length per worker required")
        k = int(klens.max()) if n else 2
    else:
        k = int(key_length)
    if keys.shape[0] != n:
        raise ValueError("one Philox key per worker required")
    sk = None if skips is None else np.ascontiguousarray(skips, dtype=np.uint64).reshape(-1)
    devs = devices_ or devices()

    def run(dev, lo, hi):
        m = hi - lo
        out = ClimbResult(
            scores=np.empty(m, dtype=np.float64),
            keys=np.empty((m, k), dtype=np.uint8),
            group_best=np.empty(m // group_size, dtype=np.int64) if group_size > 0 else None,
            draws_used=np.empty(m, dtype=np.uint64) if draws_used else None,
            last_accept=np.empty(m, dtype=np.int64) if last_accept else None,
            tries_done=np.empty(m, dtype=np.int64) if tries_done else None,
            launches=0,
        )
        if m == 0:
            return out
        c_of = np.ascontiguousarray(cof[lo:hi])
        kk = np.ascontiguousarray(keys[lo:hi])
        s = None if sk is None else np.ascontiguousarray(sk[lo:hi])
        a = _lib.SctClimbArgs()
        a.ciphers, a.offsets, a.n_ciphers = _lib.ptr(flat), _lib.ptr(off), off.size - 1
        a.cipher_of, a.keys, a.skips = _lib.ptr(c_of), _lib.ptr(kk), _lib.ptr(s)
        a.n_workers, a.key_length, a.climbings = m, k, int(climbings)
        a.p1, a.p2, a.op1_hop, a.op2_hop = int(p1), int(p2), int(op1_hop), int(op2_hop)
        a.logs, a.scores, a.keys_out = _lib.ptr(lg), _lib.ptr(out.scores), _lib.ptr(out.keys)
        a.draws_used, a.last_accept = _lib.ptr(out.draws_used), _lib.ptr(out.last_accept)
        a.tries_done = _lib.ptr(out.tries_done)
        a.group_size, a.group_best = int(group_size), _lib.ptr(out.group_best)
        a.order = int(order)
        a.flags = ((0 if speculate else _lib.FLAG_SCT_NO_SPEC)
                   | (_lib.FLAG_SCT_SPEC_REPLAY if speculate == "replay" else 0)
                   | _lib.SCT_KERNEL_FLAGS[kernel]
                   | (_lib.FLAG_SCT_TABLE_L2 if table_l2 else 0))
        kl = None if klens is None else np.ascontiguousarray(klens[lo:hi])
        a.key_lengths = _lib.ptr(kl)
        ctx = _lib.context(dev)
        with ctx.lock:
            before = ctx.launches()
            _lib.check(_lib.load().ccg_sct_climb(ctx.handle, a), "sct_climb")
            out.launches = ctx.launches() - before
        return out

    parts = _run_sharded(n, group_size, devs, run)
    return ClimbResult(
        scores=_concat(parts, "scores"), keys=_concat(parts, "keys"),
        group_best=_concat(parts, "group_best"), draws_used=_concat(parts, "draws_used"),
        last_accept=_concat(parts, "last_accept"), tries_done=_concat(parts, "tries_done"),
        launches=sum(p.launches for p in parts),
    )


def sct_fast_climb(ciphers, cipher_of, keys, table, key_length, climbings, *, p1=33, p2=66,
                   op1_hop=3, op2_hop=3, skips=None, group_size=0, draws_used=False,
                   last_accept=False, tries_done=False, lookups=True, table_l2=False,
                   window_tables=True, devices_=None) -> ClimbResult:
    """The opt-in fast SCT mode (ccg_sct_fast_climb): sct_worker (sct.py:148-170) with the
    fitness replaced by the integer sum of a quantised log table (ngrams.quantize_sct_table:
    `table` is a QuantizedSctTable or its int32[26**order] entries plus `order` attribute),
    scored incrementally over the windows of the columns a candidate moves.  Same draws,
    operators and strict acceptance as the reference; scores come back as int64 quantised
    fitness.  `lookups` reports the table lookups each worker's incremental rescoring made.
    On regular grids (text length a multiple of k, orders 2-3) a changed window is one read of
    a per-(ciphertext, k) table of window sums by column ranks; window_tables=False walks the
    window's column instead (identical results)."""
    flat, off = _lib.ragged(ciphers)
    cof = np.ascontiguousarray(cipher_of, dtype=np.int32).reshape(-1)
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, 2)
    order = int(getattr(table, "order", 0)) or {676: 2, 17576: 3, 456976: 4}.get(np.size(table), 0)
    tab = np.ascontiguousarray(getattr(table, "table", table), dtype=np.int32).reshape(-1)
    if order not in (2, 3, 4) or tab.size != 26**order:
        raise ValueError("the fast SCT table must have 26**order int32 entries, order 2..4")
    n = cof.size
    klens = None
    if np.ndim(key_length):
        klens = np.ascontiguousarray(key_length, dtype=np.int32).reshape(-1)
        if klens.size != n:
            raise ValueError("one key length per worker required")
        k = int(klens.max()) if n else 2
    else:
        k = int(key_length)
    if keys.shape[0] != n:
        raise ValueError("one Philox key per worker required")
    sk = None if skips is None else np.ascontiguousarray(skips, dtype=np.uint64).reshape(-1)
    devs = devices_ or devices()

    def run(dev, lo, hi):
        m = hi - lo
        out = ClimbResult(
            scores=np.empty(m, dtype=np.int64), keys=np.empty((m, k), dtype=np.uint8),
            group_best=np.empty(m // group_size, dtype=np.int64) if group_size > 0 else None,
            draws_used=np.empty(m, dtype=np.uint64) if draws_used else None,
            last_accept=np.empty(m, dtype=np.int64) if last_accept else None,
            tries_done=np.empty(m, dtype=np.int64) if tries_done else None, launches=0,
            lookups=np.empty(m, dtype=np.int64) if lookups else None)
        if m == 0:
            return out
        c_of = np.ascontiguousarray(cof[lo:hi])
        kk = np.ascontiguousarray(keys[lo:hi])
        s = None if sk is None else np.ascontiguousarray(sk[lo:hi])
        kl = None if klens is None else np.ascontiguousarray(klens[lo:hi])
        a = _lib.SctFastArgs()
        a.ciphers, a.offsets, a.n_ciphers = _lib.ptr(flat), _lib.ptr(off), off.size - 1
        a.cipher_of, a.keys, a.skips = _lib.ptr(c_of), _lib.ptr(kk), _lib.ptr(s)
        a.n_workers, a.key_length, a.climbings = m, k, int(climbings)
        a.p1, a.p2, a.op1_hop, a.op2_hop = int(p1), int(p2), int(op1_hop), int(op2_hop)
        a.order, a.table = order, _lib.ptr(tab)
        a.scores, a.keys_out = _lib.ptr(out.scores), _lib.ptr(out.keys)
        a.draws_used, a.last_accept = _lib.ptr(out.draws_used), _lib.ptr(out.last_accept)
        a.tries_done = _lib.ptr(out.tries_done)
        a.group_size, a.group_best = int(group_size), _lib.ptr(out.group_best)
        a.key_lengths, a.lookups = _lib.ptr(kl), _lib.ptr(out.lookups)
        a.flags = ((_lib.FLAG_SCT_TABLE_L2 if table_l2 else 0)
                   | (0 if window_tables else _lib.FLAG_SCT_NO_WINDOW_TABLES))
        ctx = _lib.context(dev)
        with ctx.lock:
            before = ctx.launches()
            _lib.check(_lib.load().ccg_sct_fast_climb(ctx.handle, a), "sct_fast_climb")
            out.launches = ctx.launches() - before
        return out

    parts = _run_sharded(n, group_size, devs, run)
    return ClimbResult(
        scores=_concat(parts, "scores"), keys=_concat(parts, "keys"),
        group_best=_concat(parts, "group_best"), draws_used=_concat(parts, "draws_used"),
        last_accept=_concat(parts, "last_accept"), tries_done=_concat(parts, "tries_done"),
        launches=sum(p.launches for p in parts), lookups=_concat(parts, "lookups"),
    )


def mas_delta_batch(texts, pairs, table_scores) -> np.ndarray:
    """text_swap_delta (mas.py:315-317) for many (text, a, b) on the GPU."""
    flat, off = _lib.ragged(texts)
    ab = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
    table = np.ascontiguousarray(table_scores, dtype=np.int64)
    out = np.empty(off.size - 1, dtype=np.int64)
    ctx = _lib.context(default_device())
    with ctx.lock:
        _lib.check(_lib.load().ccg_mas_delta_batch(ctx.handle, _lib.ptr(flat), _lib.ptr(off),
                                                   out.size, _lib.ptr(ab), _lib.ptr(table),
                                                   _lib.ptr(out)), "mas_delta")
    return out


def mas_delta_counts_batch(counts, pairs, score_matrix) -> np.ndarray:
    """swap_delta (mas.py:181-210) for many (count matrix, a, b) on the GPU."""
    cm = np.ascontiguousarray(counts, dtype=np.int64).reshape(-1, 676)
    ab = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
    sm = np.ascontiguousarray(score_matrix, dtype=np.int64).reshape(676)
    out = np.empty(cm.shape[0], dtype=np.int64)
    ctx = _lib.context(default_device())
    with ctx.lock:
        _lib.check(_lib.load().ccg_mas_delta_counts_batch(ctx.handle, _lib.ptr(cm), out.size,
                                                          _lib.ptr(ab), _lib.ptr(sm),
                                                          _lib.ptr(out)), "mas_delta_counts")
    return out


def sct_score_batch(ciphers, cipher_of, keys, logs, order=2) -> np.ndarray:
    """candidate_score (sct.py:158-160) for many (ciphertext, key) pairs on the GPU."""
    flat, off = _lib.ragged(ciphers)
    cof = np.ascontiguousarray(cipher_of, dtype=np.int32).reshape(-1)
    kk = np.ascontiguousarray(keys, dtype=np.uint8)
    if kk.ndim != 2 or kk.shape[0] != cof.size:
        raise ValueError("keys must be [n_keys, key_length]")
    lg = np.ascontiguousarray(logs, dtype=np.float64).reshape(-1)
    if lg.size != 26**int(order):
        raise ValueError(f"expected {26**int(order)} log-table entries for order {order}")
    out = np.empty(cof.size, dtype=np.float64)
    ctx = _lib.context(default_device())
    with ctx.lock:
        _lib.check(_lib.load().ccg_sct_score_ngram_batch(ctx.handle, _lib.ptr(flat), _lib.ptr(off),
                                                         off.size - 1, _lib.ptr(cof), _lib.ptr(kk),
                                                         kk.shape[1], cof.size, int(order),
                                                         _lib.ptr(lg), _lib.ptr(out)), "sct_score")
    return out


def ngram_log_score_batch(texts, order, logs) -> np.ndarray:
    """log_score_text (ngrams.py:166-172) generalised to order-n windows, bit-exact numpy
    pairwise order, on the GPU."""
    flat, off = _lib.ragged(texts)
    lg = np.ascontiguousarray(logs, dtype=np.float64).reshape(-1)
    if lg.size != 26**int(order):
        raise ValueError(f"expected {26**int(order)} log-table entries for order {order}")
    out = np.empty(off.size - 1, dtype=np.float64)
    ctx = _lib.context(default_device())
    with ctx.lock:
        _lib.check(_lib.load().ccg_ngram_log_score_batch(ctx.handle, _lib.ptr(flat), _lib.ptr(off),
                                                         off.size - 1, int(order), _lib.ptr(lg),
                                                         _lib.ptr(out)), "ngram_log_score")
    return out


def mas_det_step_batch(texts, pivots, table_scores) -> np.ndarray:
    """All 325 pair-worker scores of deterministic_step (mas.py:84-120) for many
    (text, pivot) on the GPU: int64[n, 325]."""
    flat, off = _lib.ragged(texts)
    pv = np.ascontiguousarray(pivots, dtype=np.int32).reshape(-1, 2)
    table = np.ascontiguousarray(table_scores, dtype=np.int64)
    out = np.empty((off.size - 1, 325), dtype=np.int64)
    ctx = _lib.context(default_device())
    with ctx.lock:
        _lib.check(_lib.load().ccg_mas_det_step_batch(ctx.handle, _lib.ptr(flat), _lib.ptr(off),
                                                      off.size - 1, _lib.ptr(pv), _lib.ptr(table),
                                                      _lib.ptr(out)), "det_step")
    return out


def bench_smem_bandwidth(device=None) -> float:
    """Measured conflict-free LDS bandwidth of the device, bytes/s (roofline denominator)."""
    import ctypes as C

    out = C.c_double(0.0)
    ctx = _lib.context(default_device() if device is None else device)
    with ctx.lock:
        _lib.check(_lib.load().ccg_bench_smem_bandwidth(ctx.handle, C.byref(out)), "smem bench")
    return out.value


def bench_l2_gather(entries: int = 26**4, device=None) -> float:
    """Measured random uint16 gathers/s from an L2-resident table of `entries` entries (the
    quadgram table by default): the roofline denominator of the n-gram climb at order 4."""
    import ctypes as C

    out = C.c_double(0.0)
    ctx = _lib.context(default_device() if device is None else device)
    with ctx.lock:
        _lib.check(_lib.load().ccg_bench_l2_gather(ctx.handle, int(entries), C.byref(out)),
                   "L2 gather bench")
    return out.value


class JobHistories(collections.abc.Sequence):
    """Per-job [(iteration, score), ...] lists of a mas_det_solve batch, built on access:
    turning every history of a 20,000-job batch into Python tuples up front would cost more
    than the solve itself."""

    def __init__(self, parts=()):
        # (iterations, scores, offsets): job j's entries at [offsets[j], offsets[j+1])
        self._parts = [p for p in parts if p[2].size > 1]
        self._ends = np.cumsum([p[2].size - 1 for p in self._parts]).tolist()

    def __len__(self):
        return self._ends[-1] if self._ends else 0

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("job index out of range")
        k = bisect.bisect_right(self._ends, i)
        it, sc, off = self._parts[k]
        j = i - (self._ends[k - 1] if k else 0)
        lo, hi = int(off[j]), int(off[j + 1])
        return list(zip(it[lo:hi].tolist(), sc[lo:hi].tolist()))

    def __eq__(self, other):
        return len(self) == len(other) and all(a == b for a, b in zip(self, other))


@dataclass
class DetResult:
    scores: np.ndarray          # int64 per job
    maps: np.ndarray            # uint8[n, 26] cipher letter -> plaintext letter
    history: JobHistories       # per job: [(iteration, score), ...] (built on access)
    draws_used: np.ndarray
    launches: int


def mas_det_solve(ciphers, cipher_of, keys, table_scores, iterations, *, devices_=None) -> DetResult:
    """solve_deterministic (mas.py:140-169) for a batch of jobs, one CTA each, the whole
    iteration loop on the device.  keys: uint64[n, 2] PIVOT-stream Philox keys."""
    flat, off = _lib.ragged(ciphers)
    cof = np.ascontiguousarray(cipher_of, dtype=np.int32).reshape(-1)
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, 2)
    table = np.ascontiguousarray(table_scores, dtype=np.int64)
    n, it = cof.size, int(iterations)
    if keys.shape[0] != n:
        raise ValueError("one Philox key per job required")
    devs = devices_ or devices()

    def run(dev, lo, hi):
        m = hi - lo
        out = DetResult(scores=np.empty(m, dtype=np.int64), maps=np.empty((m, 26), dtype=np.uint8),
                        history=JobHistories(), draws_used=np.empty(m, dtype=np.uint64), launches=0)
        if m == 0:
            return out
        # packed histories: capacity m * iterations, but only the accepts' pages are touched
        hi_it = np.empty(m * max(1, it), dtype=np.int32)
        hi_sc = np.empty(m * max(1, it), dtype=np.int64)
        hl = np.empty(m, dtype=np.int32)
        hoff = np.zeros(m + 1, dtype=np.int64)
        c_of = np.ascontiguousarray(cof[lo:hi])
        k = np.ascontiguousarray(keys[lo:hi])
        a = _lib.MasDetArgs()
        a.ciphers, a.offsets, a.n_ciphers = _lib.ptr(flat), _lib.ptr(off), off.size - 1
        a.cipher_of, a.keys, a.n_jobs, a.iterations = _lib.ptr(c_of), _lib.ptr(k), m, it
        a.table, a.scores, a.maps = _lib.ptr(table), _lib.ptr(out.scores), _lib.ptr(out.maps)
        a.hist_iter, a.hist_score, a.hist_len = _lib.ptr(hi_it), _lib.ptr(hi_sc), _lib.ptr(hl)
        a.draws_used = _lib.ptr(out.draws_used)
        a.hist_offsets = _lib.ptr(hoff)
        ctx = _lib.context(dev)
        with ctx.lock:
            before = ctx.launches()
            _lib.check(_lib.load().ccg_mas_det_solve(ctx.handle, a), "mas_det_solve")
            out.launches = ctx.launches() - before
        out.history = JobHistories([(hi_it, hi_sc, hoff)])
        return out

    parts = _run_sharded(n, 0, devs, run)
    return DetResult(scores=np.concatenate([p.scores for p in parts]),
                     maps=np.concatenate([p.maps for p in parts]),
                     history=JobHistories([q for p in parts for q in p.history._parts]),
                     draws_used=np.concatenate([p.draws_used for p in parts]),
                     launches=sum(p.launches for p in parts))


def ngram_score_batch(texts, order, table_scores) -> np.ndarray:
    """Integer n-gram fitness (ngrams.py:134-140 generalised to order-n windows) on the GPU."""
    flat, off = _lib.ragged(texts)
    table = np.ascontiguousarray(table_scores, dtype=np.int64).reshape(-1)
    if table.size != 26**int(order):
        raise ValueError(f"expected {26**int(order)} table entries")
    out = np.empty(off.size - 1, dtype=np.int64)
    ctx = _lib.context(default_device())
    with ctx.lock:
        _lib.check(_lib.load().ccg_ngram_score_batch(ctx.handle, _lib.ptr(flat), _lib.ptr(off),
                                                     off.size - 1, int(order), _lib.ptr(table),
                                                     _lib.ptr(out)), "ngram_score")
    return out
