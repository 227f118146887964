#!/usr/bin/env python
"""Where the bench's end-to-end time goes: the device-resident step (ccg_mas_climb_dev), the
host-buffer C call (ccg_mas_climb from pinned buffers) and the Python engine.mas_climb
around it, all host-timed with a synchronize, on the bench workload.

Measured (r1): 85.7 ms device-resident, 87.7 ms through the C call, +0.1 ms in Python.  A
four-chunk upload/climb/download pipeline on two streams measured 88.5 ms: the persistent
kernels of consecutive chunks cannot overlap until whole blocks retire, which costs what the
hidden copies save."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2103_13937_b200 import _lib, engine  # noqa: E402

n_c = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
W, K = 64, 10_000
plains, ciphers, scores, lengths = bench.make_workload(n_c, 0)
keys = bench.worker_keys(n_c, W, 0)
flat, off = _lib.ragged(ciphers)
cof = np.repeat(np.arange(n_c, dtype=np.int32), W)
n = n_c * W
ctx = _lib.context(0)
L = _lib.load()


def pinned(arr):
    p = C.c_void_p()
    _lib.check(L.ccg_host_alloc(arr.nbytes, C.byref(p)), "host_alloc")
    out = np.frombuffer((C.c_uint8 * arr.nbytes).from_address(p.value), dtype=arr.dtype)
    out = out.reshape(arr.shape)
    out[...] = arr
    return out


p_flat, p_off, p_cof, p_keys = pinned(flat), pinned(off), pinned(cof), pinned(keys)
p_scores, p_maps = pinned(np.zeros(n, np.int64)), pinned(np.zeros((n, 26), np.uint8))
p_best = pinned(np.zeros(n_c, np.int64))
tab = np.ascontiguousarray(scores, dtype=np.int64)


def host_args():
    a = _lib.MasClimbArgs()
    a.ciphers, a.offsets, a.n_ciphers = _lib.ptr(p_flat), _lib.ptr(p_off), n_c
    a.cipher_of, a.keys, a.skips = _lib.ptr(p_cof), _lib.ptr(p_keys), None
    a.n_workers, a.climbings, a.table = n, K, _lib.ptr(tab)
    a.scores, a.maps = _lib.ptr(p_scores), _lib.ptr(p_maps)
    a.group_size, a.group_best = W, _lib.ptr(p_best)
    a.flags = 0
    return a


def dev(arr):
    p = ctx.dev_alloc(max(1, arr.nbytes))
    ctx.h2d(p, np.ascontiguousarray(arr))
    return p


d = _lib.MasClimbArgs()
d.ciphers, d.offsets, d.n_ciphers = dev(flat), dev(off), n_c
d.cipher_of, d.keys, d.skips = dev(cof), dev(keys), None
d.n_workers, d.climbings, d.table = n, K, dev(tab)
d.scores, d.maps = ctx.dev_alloc(n * 8), ctx.dev_alloc(n * 26)
d.group_size, d.group_best = W, ctx.dev_alloc(n_c * 8)
d.max_len, d.table_max = int(lengths.max()), int(tab.max())
d.flags = 0
ctx.synchronize()


def timeit(fn, reps=3):
    fn()
    ctx.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ctx.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)


a = host_args()
t_dev = timeit(lambda: _lib.check(L.ccg_mas_climb_dev(ctx.handle, d), "dev"))
t_c = timeit(lambda: _lib.check(L.ccg_mas_climb(ctx.handle, a), "host"))
batch = _lib.Packed.__new__(_lib.Packed)
batch.flat, batch.offsets = p_flat, p_off
res = engine.ClimbResult(scores=p_scores, keys=p_maps, group_best=p_best, draws_used=None,
                         last_accept=None, tries_done=None, launches=0)
t_py = timeit(lambda: engine.mas_climb(batch, p_cof, p_keys, tab, K, group_size=W, out=res))
print(f"device-resident {t_dev:.2f} ms | C host call {t_c:.2f} ms | engine.mas_climb {t_py:.2f} ms")
