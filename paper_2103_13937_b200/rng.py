"""Per-worker counter-based random streams (reference rng.py:1-102).

Worker w of restart r draws from numpy's Philox4x64-10 keyed [seed, (r << 32) | w]
(rng.py:27-33, 58-64).  The GPU kernels regenerate exactly that stream on device
(csrc/ccg_rng.cuh); this module holds the stream bookkeeping and the host-facing
WorkerRng, whose draws are also produced by the GPU (ccg_philox_uniform) in blocks of
4096, like the reference's buffering (rng.py:19, 68-75).
"""
from __future__ import annotations

import numpy as np

from . import _lib

_BUFFER = 4096
PIVOT_STREAM = 2**32 - 1
KEYGEN_STREAM = 2**32 - 2


def worker_stream_index(restart: int, worker: int) -> int:
    if restart < 0 or worker < 0:
        raise ValueError("restart and worker must be non-negative")
    if worker >= KEYGEN_STREAM:
        raise ValueError(f"worker index must be below {KEYGEN_STREAM}")
    return (restart << 32) | worker


def pivot_stream_index(restart: int) -> int:
    if restart < 0:
        raise ValueError("restart must be non-negative")
    return (restart << 32) | PIVOT_STREAM


def uniform_to_int(u: float, bound: int) -> int:
    if bound < 1:
        raise ValueError("bound must be at least 1")
    return int(u * bound)


def _through_float64(v: int) -> int:
    f = float(v)  # round to nearest double, as numpy's int->float64 promotion does
    return 0 if f >= 2.0**64 else int(f)  # 2**64 does not fit uint64: numpy's cast yields 0


def philox_key(seed: int, stream: int) -> tuple[int, int]:
    """The (k0, k1) Philox key numpy actually installs for WorkerRng(seed, stream).

    rng.py:63-64 passes the list [seed % 2**64, stream % 2**64]; numpy converts it with
    np.asarray(...).astype(uint64).  A list mixing a value >= 2**63 (uint64 class) with
    one below (int64 class) is promoted to float64 first, so both words are rounded to
    doubles.  Reproducing this keeps every stream bit-identical to the reference."""
    s, w = int(seed) % 2**64, int(stream) % 2**64
    if (s >= 2**63) != (w >= 2**63):
        s, w = _through_float64(s), _through_float64(w)
    return s, w


def philox_keys(seeds, streams) -> np.ndarray:
    """uint64[n, 2] keys for parallel arrays of seeds and stream indices."""
    seeds = np.asarray(seeds, dtype=object).reshape(-1)
    streams = np.asarray(streams, dtype=object).reshape(-1)
    if seeds.size == 1 and streams.size > 1:
        seeds = np.repeat(seeds, streams.size)
    out = np.empty((streams.size, 2), dtype=np.uint64)
    for i, (s, w) in enumerate(zip(seeds.tolist(), streams.tolist())):
        out[i] = philox_key(s, w)
    return out


def draws(seed: int, stream: int, count: int, skip: int = 0, device: int | None = None) -> np.ndarray:
    """`count` uniforms of stream (seed, stream) after `skip` draws, generated on the GPU."""
    from .engine import default_device

    k0, k1 = philox_key(seed, stream)
    out = np.empty(int(count), dtype=np.float64)
    ctx = _lib.context(default_device() if device is None else device)
    with ctx.lock:
        _lib.check(_lib.load().ccg_philox_uniform(ctx.handle, k0, k1, int(skip), out.size,
                                                  _lib.ptr(out)), "philox_uniform")
    return out


class WorkerRng:
    """One worker's private stream (rng.py:50-97).

    `position` counts the draws consumed so far; GPU workers started from this object
    begin at `position` and advance it by the draws they used, exactly as the
    reference's in-process worker would have advanced its generator."""

    def __init__(self, global_seed: int, worker_index: int):
        if worker_index < 0:
            raise ValueError("worker_index must be non-negative")
        self.global_seed = int(global_seed)
        self.worker_index = int(worker_index)
        self.key = philox_key(self.global_seed, self.worker_index)
        self.position = 0
        self._buf = np.empty(0, dtype=np.float64)
        self._buf_start = 0

    def advance(self, new_position: int) -> None:
        self.position = int(new_position)

    def next_uniform(self) -> float:
        i = self.position - self._buf_start
        if not 0 <= i < self._buf.size:
            self._buf = draws(self.global_seed, self.worker_index, _BUFFER, skip=self.position)
            self._buf_start = self.position
            i = 0
        self.position += 1
        return float(self._buf[i])

    def next_int_below(self, bound: int) -> int:
        return uniform_to_int(self.next_uniform(), bound)

    def next_distinct_pair(self, bound: int) -> tuple[int, int]:
        if bound < 2:
            raise ValueError("bound must be at least 2 for a distinct pair")
        a = self.next_int_below(bound)
        b = self.next_int_below(bound)
        while b == a:
            b = self.next_int_below(bound)
        return a, b

    def permutation(self, n: int) -> np.ndarray:
        perm = np.arange(n, dtype=np.int64)
        for i in range(n - 1, 0, -1):
            j = self.next_int_below(i + 1)
            perm[[i, j]] = perm[[j, i]]
        return perm


def init_worker_state(global_seed: int, worker_index: int) -> WorkerRng:
    return WorkerRng(global_seed, worker_index)
