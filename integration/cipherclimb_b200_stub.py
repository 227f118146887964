"""The reference-side binding of INTEGRATION.md section 2: the file a maintainer drops into
the reference package as `cipherclimb/_b200.py` to keep `cipherclimb` and replace only its
worker pool (search.py:49-58 run_worker_pool) with one C call per batch.

It depends on ctypes and numpy only -- nothing from this repo's Python package -- and binds
the C ABI of include/cipherclimb_b200.h directly.  tests/test_integration_stub.py runs it on
reference-shaped task tuples (mas.py:266-270, sct.py:194-198) and checks the reference's own
solve outputs frozen in tests/golden/.

The one-line changes in the reference:
    mas.py:272  outcomes = run_worker_pool(_stochastic_task, tasks, jobs=jobs)
             -> outcomes = _b200.run_stochastic_pool(tasks)
    sct.py:199  outcomes = run_worker_pool(_sct_task, tasks, jobs=jobs)
             -> outcomes = _b200.run_sct_pool(tasks)
"""
import ctypes as C
import os

import numpy as np

_P, _i64, _i32, _u32 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32
_lib = None
_ctx = C.c_void_p()


class MasClimbArgs(C.Structure):  # include/cipherclimb_b200.h ccg_mas_climb_args
    _fields_ = [("ciphers", _P), ("offsets", _P), ("n_ciphers", _i64), ("cipher_of", _P),
                ("keys", _P), ("skips", _P), ("n_workers", _i64), ("climbings", _i64),
                ("table", _P), ("scores", _P), ("maps", _P), ("draws_used", _P),
                ("last_accept", _P), ("tries_done", _P), ("group_size", _i32),
                ("group_best", _P), ("max_len", _i64), ("table_max", _i64), ("flags", _u32),
                ("accepts", _P)]


class SctClimbArgs(C.Structure):  # include/cipherclimb_b200.h ccg_sct_climb_args
    _fields_ = [("ciphers", _P), ("offsets", _P), ("n_ciphers", _i64), ("cipher_of", _P),
                ("keys", _P), ("skips", _P), ("n_workers", _i64), ("key_length", _i32),
                ("climbings", _i64), ("p1", _i32), ("p2", _i32), ("op1_hop", _i32),
                ("op2_hop", _i32), ("logs", _P), ("scores", _P), ("keys_out", _P),
                ("draws_used", _P), ("last_accept", _P), ("tries_done", _P),
                ("group_size", _i32), ("group_best", _P), ("text_len", _i64), ("flags", _u32),
                ("order", _i32), ("key_lengths", _P)]


def load(path=None, device=0):
    """Open libcipherclimb_b200.so (built by the engine's __graft_entry__.build()) and a
    context on `device`."""
    global _lib
    if _lib is None:
        _lib = C.CDLL(path or os.environ.get("CCG_LIB", "libcipherclimb_b200.so"))
        _lib.ccg_last_error.restype = C.c_char_p
        _lib.ccg_ctx_create.argtypes = [C.c_int, _P]
        _lib.ccg_mas_climb.argtypes = [_P, C.POINTER(MasClimbArgs)]
        _lib.ccg_sct_climb.argtypes = [_P, C.POINTER(SctClimbArgs)]
        if _lib.ccg_ctx_create(int(device), C.byref(_ctx)) != 0:
            raise RuntimeError(_lib.ccg_last_error().decode())
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _philox_keys(tasks):
    # numpy's key for WorkerRng(seed, stream), rng.py:63-64: np.asarray([...]).astype(uint64)
    # (a list mixing a value >= 2^63 with a smaller one goes through float64, as in numpy)
    return np.array([np.asarray([t[-2] % 2**64, t[-1] % 2**64]).astype(np.uint64) for t in tasks],
                    dtype=np.uint64)


def _check(rc):
    if rc != 0:
        raise RuntimeError(_lib.ccg_last_error().decode())


def run_stochastic_pool(tasks):
    """run_worker_pool(_stochastic_task, tasks) (mas.py:247-250, 272): tasks[i] =
    (cipher, scores, climbings, seed, stream); returns [(text, score)] in task order."""
    load()
    cipher, scores, climbings = tasks[0][0], tasks[0][1], tasks[0][2]
    text = np.ascontiguousarray(cipher, dtype=np.uint8)
    off = np.array([0, text.size], dtype=np.int64)
    keys = _philox_keys(tasks)
    n = len(tasks)
    out_s = np.empty(n, np.int64)
    out_m = np.empty((n, 26), np.uint8)
    table = np.ascontiguousarray(scores, np.int64)
    a = MasClimbArgs(ciphers=_p(text), offsets=_p(off), n_ciphers=1,
                     cipher_of=_p(np.zeros(n, np.int32)), keys=_p(keys), n_workers=n,
                     climbings=int(climbings), table=_p(table), scores=_p(out_s),
                     maps=_p(out_m), max_len=text.size, table_max=int(table.max()))
    _check(_lib.ccg_mas_climb(_ctx, C.byref(a)))
    cipher = np.asarray(cipher, dtype=np.int64)
    return [(out_m[i].astype(np.int64)[cipher], int(out_s[i])) for i in range(n)]


def run_sct_pool(tasks):
    """run_worker_pool(_sct_task, tasks) (sct.py:173-176, 199): tasks[i] =
    (cipher, logs, floor, cfg, seed, stream); returns [(key, score)] in task order."""
    load()
    cipher, logs, cfg = tasks[0][0], tasks[0][1], tasks[0][3]
    text = np.ascontiguousarray(cipher, dtype=np.uint8)
    off = np.array([0, text.size], dtype=np.int64)
    keys = _philox_keys(tasks)
    n, k = len(tasks), int(cfg.key_length)
    out_s = np.empty(n, np.float64)
    out_k = np.empty((n, k), np.uint8)
    lg = np.ascontiguousarray(logs, np.float64)
    a = SctClimbArgs(ciphers=_p(text), offsets=_p(off), n_ciphers=1,
                     cipher_of=_p(np.zeros(n, np.int32)), keys=_p(keys), n_workers=n,
                     key_length=k, climbings=int(cfg.climbings), p1=int(cfg.p1),
                     p2=int(cfg.p2), op1_hop=int(cfg.op1_hop), op2_hop=int(cfg.op2_hop),
                     logs=_p(lg), scores=_p(out_s), keys_out=_p(out_k), text_len=text.size,
                     order=2)
    _check(_lib.ccg_sct_climb(_ctx, C.byref(a)))
    return [(out_k[i].astype(np.int64), float(out_s[i])) for i in range(n)]
