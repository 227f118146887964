"""ctypes binding of libcipherclimb_b200.so (C ABI: include/cipherclimb_b200.h).

This is the only path from the Python API to the GPU.  There is no CPU fallback: if the
shared library is missing or no sm_100 device is visible, every solver raises
EngineError.  Build the library with `python -c "import __graft_entry__ as g; g.build()"`
(or `make -C paper_2103_13937_b200/csrc`).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libcipherclimb_b200.so"
ABI_VERSION = 1
ALPHA = 26

CCG_OK, CCG_ERR_INVALID, CCG_ERR_CUDA, CCG_ERR_NO_DEVICE, CCG_ERR_UNSUPPORTED = 0, -1, -2, -3, -4
FLAG_EARLY_EXIT = 1
FLAG_SCT_NO_SPEC = 0x100  # SCT: never use the speculative latency kernels
FLAG_SCT_KERNEL_WARP = 0x200  # SCT: one warp per worker instead of one lane per worker
FLAG_SCT_TABLE_L2 = 0x400  # SCT lane kernel: trigram table read through L2, not shared memory
FLAG_SCT_KERNEL_LANE = 0x800  # SCT: one worker per lane
FLAG_SCT_SPEC_REPLAY = 0x1000  # SCT latency mode: per-round draw replay instead of the parsed chain
FLAG_SCT_NO_WINDOW_TABLES = 0x2000  # SCT fast mode: no regular-grid window-sum tables
SCT_KERNEL_FLAGS = {"auto": 0, "lane": FLAG_SCT_KERNEL_LANE, "warp": FLAG_SCT_KERNEL_WARP}
KERNEL_FLAGS = {"auto": 0, "dform": 0x10, "tform": 0x20, "packed": 0x30, "dtable": 0x40}


class EngineError(RuntimeError):
    """The CUDA engine could not run (library missing, no device, CUDA error, limit)."""


_P = C.c_void_p
_i64, _u64, _i32, _u32 = C.c_int64, C.c_uint64, C.c_int32, C.c_uint32


class MasClimbArgs(C.Structure):
    _fields_ = [
        ("ciphers", _P), ("offsets", _P), ("n_ciphers", _i64), ("cipher_of", _P), ("keys", _P),
        ("skips", _P), ("n_workers", _i64), ("climbings", _i64), ("table", _P),
        ("scores", _P), ("maps", _P), ("draws_used", _P), ("last_accept", _P),
        ("tries_done", _P), ("group_size", _i32), ("group_best", _P), ("max_len", _i64),
        ("table_max", _i64), ("flags", _u32), ("accepts", _P),
    ]


class SctClimbArgs(C.Structure):
    _fields_ = [
        ("ciphers", _P), ("offsets", _P), ("n_ciphers", _i64), ("cipher_of", _P), ("keys", _P),
        ("skips", _P), ("n_workers", _i64), ("key_length", _i32), ("climbings", _i64),
        ("p1", _i32), ("p2", _i32), ("op1_hop", _i32), ("op2_hop", _i32), ("logs", _P),
        ("scores", _P), ("keys_out", _P), ("draws_used", _P), ("last_accept", _P),
        ("tries_done", _P), ("group_size", _i32), ("group_best", _P), ("text_len", _i64),
        ("flags", _u32), ("order", _i32), ("key_lengths", _P),
    ]


class SctFastArgs(C.Structure):
    _fields_ = [
        ("ciphers", _P), ("offsets", _P), ("n_ciphers", _i64), ("cipher_of", _P), ("keys", _P),
        ("skips", _P), ("n_workers", _i64), ("key_length", _i32), ("climbings", _i64),
        ("p1", _i32), ("p2", _i32), ("op1_hop", _i32), ("op2_hop", _i32), ("order", _i32),
        ("table", _P), ("scores", _P), ("keys_out", _P), ("draws_used", _P),
        ("last_accept", _P), ("tries_done", _P), ("group_size", _i32), ("group_best", _P),
        ("key_lengths", _P), ("lookups", _P), ("flags", _u32),
    ]


class MasNgramArgs(C.Structure):
    _fields_ = [
        ("ciphers", _P), ("offsets", _P), ("n_ciphers", _i64), ("cipher_of", _P), ("keys", _P),
        ("skips", _P), ("n_workers", _i64), ("climbings", _i64), ("order", _i32), ("table", _P),
        ("scores", _P), ("maps", _P), ("draws_used", _P), ("last_accept", _P),
        ("tries_done", _P), ("group_size", _i32), ("group_best", _P), ("max_len", _i64),
        ("flags", _u32), ("computed", _P), ("lookups", _P),
    ]


class MasDetArgs(C.Structure):
    _fields_ = [
        ("ciphers", _P), ("offsets", _P), ("n_ciphers", _i64), ("cipher_of", _P), ("keys", _P),
        ("n_jobs", _i64), ("iterations", _i64), ("table", _P), ("scores", _P), ("maps", _P),
        ("hist_iter", _P), ("hist_score", _P), ("hist_len", _P), ("draws_used", _P),
        ("max_len", _i64), ("table_max", _i64), ("hist_offsets", _P),
    ]


EXPORTS = {
    # name: (restype, argtypes)
    "ccg_abi_version": (C.c_int, []),
    "ccg_last_error": (C.c_char_p, []),
    "ccg_device_count": (C.c_int, [_P]),
    "ccg_ctx_create": (C.c_int, [C.c_int, _P]),
    "ccg_ctx_destroy": (C.c_int, [_P]),
    "ccg_ctx_synchronize": (C.c_int, [_P]),
    "ccg_ctx_stream": (C.c_int, [_P, _P]),
    "ccg_ctx_device": (C.c_int, [_P, _P]),
    "ccg_ctx_launch_count": (C.c_int, [_P, _P]),
    "ccg_ctx_sm_count": (C.c_int, [_P, _P]),
    "ccg_dev_alloc": (C.c_int, [_P, C.c_size_t, _P]),
    "ccg_dev_free": (C.c_int, [_P, _P]),
    "ccg_host_alloc": (C.c_int, [C.c_size_t, _P]),
    "ccg_host_free": (C.c_int, [_P]),
    "ccg_memcpy_h2d": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "ccg_memcpy_d2h": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "ccg_philox_uniform": (C.c_int, [_P, _u64, _u64, _u64, _i64, _P]),
    "ccg_philox_int_below": (C.c_int, [_P, _u64, _u64, _u64, _u32, _i64, _P]),
    "ccg_score_text_batch": (C.c_int, [_P, _P, _P, _i64, _P, _P]),
    "ccg_log_score_text_batch": (C.c_int, [_P, _P, _P, _i64, _P, _P]),
    "ccg_mas_delta_batch": (C.c_int, [_P, _P, _P, _i64, _P, _P, _P]),
    "ccg_mas_delta_counts_batch": (C.c_int, [_P, _P, _i64, _P, _P, _P]),
    "ccg_mas_climb": (C.c_int, [_P, C.POINTER(MasClimbArgs)]),
    "ccg_mas_climb_dev": (C.c_int, [_P, C.POINTER(MasClimbArgs)]),
    "ccg_ngram_score_batch": (C.c_int, [_P, _P, _P, _i64, _i32, _P, _P]),
    "ccg_mas_ngram_climb": (C.c_int, [_P, C.POINTER(MasNgramArgs)]),
    "ccg_mas_ngram_climb_dev": (C.c_int, [_P, C.POINTER(MasNgramArgs)]),
    "ccg_mas_det_step_batch": (C.c_int, [_P, _P, _P, _i64, _P, _P, _P]),
    "ccg_mas_det_solve": (C.c_int, [_P, C.POINTER(MasDetArgs)]),
    "ccg_mas_det_solve_dev": (C.c_int, [_P, C.POINTER(MasDetArgs)]),
    "ccg_sct_score_batch": (C.c_int, [_P, _P, _P, _i64, _P, _P, _i32, _i64, _P, _P]),
    "ccg_ngram_log_score_batch": (C.c_int, [_P, _P, _P, _i64, _i32, _P, _P]),
    "ccg_sct_score_ngram_batch": (C.c_int, [_P, _P, _P, _i64, _P, _P, _i32, _i64, _i32, _P, _P]),
    "ccg_sct_climb": (C.c_int, [_P, C.POINTER(SctClimbArgs)]),
    "ccg_sct_climb_dev": (C.c_int, [_P, C.POINTER(SctClimbArgs)]),
    "ccg_sct_fast_climb": (C.c_int, [_P, C.POINTER(SctFastArgs)]),
    "ccg_encrypt_batch": (C.c_int, [_P, _i32, _P, _P, _i64, _P, _P, _i32, _P, _P]),
    "ccg_bench_smem_bandwidth": (C.c_int, [_P, _P]),
    "ccg_bench_l2_gather": (C.c_int, [_P, _i64, _P]),
}

_lib = None
_lock = threading.Lock()


def load(path: Path | None = None):
    """Load the shared library (raises EngineError if it is missing)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path or os.environ.get("CCG_LIB", LIB_PATH))
        if not p.exists():
            raise EngineError(
                f"CUDA engine library not found at {p}; build it with __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        L = C.CDLL(str(p))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.ccg_abi_version() != ABI_VERSION:
            raise EngineError(f"ABI mismatch: library {L.ccg_abi_version()}, binding {ABI_VERSION}")
        _lib = L
        return L


def check(rc: int, what: str):
    if rc != CCG_OK:
        msg = load().ccg_last_error().decode(errors="replace")
        if rc == CCG_ERR_INVALID:
            raise ValueError(msg)
        raise EngineError(f"{what}: {msg} (code {rc})")


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def device_count() -> int:
    n = C.c_int(0)
    check(load().ccg_device_count(C.byref(n)), "ccg_device_count")
    return n.value


class Context:
    """One device + one CUDA stream + grow-only HBM scratch (ccg_ctx)."""

    def __init__(self, device: int = 0):
        L = load()
        h = C.c_void_p()
        check(L.ccg_ctx_create(int(device), C.byref(h)), "ccg_ctx_create")
        self._h = h
        self.device = int(device)
        self.lock = threading.Lock()

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            load().ccg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass

    def stream(self) -> int:
        s = C.c_void_p()
        check(load().ccg_ctx_stream(self._h, C.byref(s)), "ccg_ctx_stream")
        return s.value or 0

    def launches(self) -> int:
        n = C.c_int64()
        check(load().ccg_ctx_launch_count(self._h, C.byref(n)), "ccg_ctx_launch_count")
        return n.value

    def sm_count(self) -> int:
        n = C.c_int()
        check(load().ccg_ctx_sm_count(self._h, C.byref(n)), "ccg_ctx_sm_count")
        return n.value

    def synchronize(self):
        check(load().ccg_ctx_synchronize(self._h), "ccg_ctx_synchronize")

    # ------------------------------------------------------------ device memory
    def dev_alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        check(load().ccg_dev_alloc(self._h, int(nbytes), C.byref(p)), "ccg_dev_alloc")
        return p.value

    def dev_free(self, p: int):
        check(load().ccg_dev_free(self._h, C.c_void_p(p)), "ccg_dev_free")

    def h2d(self, dst: int, src: np.ndarray):
        check(load().ccg_memcpy_h2d(self._h, C.c_void_p(dst), ptr(src), src.nbytes), "h2d")

    def d2h(self, dst: np.ndarray, src: int):
        check(load().ccg_memcpy_d2h(self._h, ptr(dst), C.c_void_p(src), dst.nbytes), "d2h")


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts.setdefault(device, ctx)
            ctx = _contexts[device]
    return ctx


class Packed:
    """A pre-packed ragged batch of letter arrays: uint8 letters + int64 offsets[n+1]
    (what every batch entry point hands to the C ABI).  Pass it instead of a list to skip
    the per-call packing."""

    def __init__(self, flat, offsets):
        self.flat = np.ascontiguousarray(flat, dtype=np.uint8)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        if self.offsets.ndim != 1 or self.offsets.size < 1 or self.offsets[0] != 0:
            raise ValueError("offsets must be int64[n+1] starting at 0")
        if self.offsets[-1] != self.flat.size or (np.diff(self.offsets) < 0).any():
            raise ValueError("offsets must be non-decreasing and end at len(flat)")
        if self.flat.size and self.flat.max() >= ALPHA:
            raise ValueError("letter indices must lie in 0..25")

    def __len__(self):
        return self.offsets.size - 1

    def __getitem__(self, i):
        return self.flat[self.offsets[i]:self.offsets[i + 1]]

    @classmethod
    def of(cls, texts) -> "Packed":
        flat, off = ragged(texts)
        p = cls.__new__(cls)
        p.flat, p.offsets = flat, off
        return p


def ragged(texts) -> tuple[np.ndarray, np.ndarray]:
    """Concatenate letter arrays into (uint8 flat, int64 offsets[n+1])."""
    if isinstance(texts, Packed):
        return texts.flat, texts.offsets
    n = len(texts)
    offsets = np.zeros(n + 1, dtype=np.int64)
    if n == 0:
        return np.zeros(0, dtype=np.uint8), offsets
    arrs = [t if isinstance(t, np.ndarray) else np.asarray(t, dtype=np.int64) for t in texts]
    offsets[1:] = np.cumsum(np.fromiter((a.size for a in arrs), dtype=np.int64, count=n))
    flat = np.concatenate([a.reshape(-1) for a in arrs]) if offsets[-1] else np.zeros(0, np.int64)
    if flat.size and (flat.min() < 0 or flat.max() >= ALPHA):
        raise ValueError("letter indices must lie in 0..25")
    return np.ascontiguousarray(flat, dtype=np.uint8), offsets
