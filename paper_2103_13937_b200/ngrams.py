"""Bigram tables and text fitness (reference ngrams.py:1-172).

Table construction, parsing and formatting are host-side.  The fitness functions
`score_text` / `log_score_text` run on the GPU through the C ABI (bit-exact: integer
sums, and float64 sums in numpy's pairwise order).
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .codec import ALPHABET_SIZE, MappedText, map_text, normalize

TABLE_SIZE = ALPHABET_SIZE * ALPHABET_SIZE  # 676
DEFAULT_LOG_FLOOR = -24.0


def bigram_index(first: int, second: int) -> int:
    if not (0 <= first < ALPHABET_SIZE and 0 <= second < ALPHABET_SIZE):
        raise ValueError(f"letter indices out of range: ({first}, {second})")
    return ALPHABET_SIZE * first + second


@dataclass(frozen=True)
class BigramTable:
    """676 non-negative integer scores indexed by 26*first + second."""

    scores: np.ndarray

    def __post_init__(self):
        arr = np.ascontiguousarray(self.scores, dtype=np.int64)
        if arr.shape != (TABLE_SIZE,):
            raise ValueError(f"expected {TABLE_SIZE} entries, got {arr.shape}")
        if arr.size and arr.min() < 0:
            raise ValueError("bigram scores must be non-negative")
        object.__setattr__(self, "scores", arr)

    @property
    def matrix(self) -> np.ndarray:
        return self.scores.reshape(ALPHABET_SIZE, ALPHABET_SIZE)


@dataclass(frozen=True)
class LogBigramTable:
    """676 log2 bigram probabilities; unseen bigrams sit at `floor`."""

    logs: np.ndarray
    floor: float

    def __post_init__(self):
        arr = np.ascontiguousarray(self.logs, dtype=np.float64)
        if arr.shape != (TABLE_SIZE,):
            raise ValueError(f"expected {TABLE_SIZE} entries, got {arr.shape}")
        if not np.isfinite(arr).all():
            raise ValueError("log scores must be finite")
        if arr.size and arr.max() > 0:
            raise ValueError("log2 probabilities cannot be positive")
        if arr.size and arr.min() < self.floor:
            raise ValueError("log table entries below the configured floor")
        object.__setattr__(self, "logs", arr)

    @property
    def matrix(self) -> np.ndarray:
        return self.logs.reshape(ALPHABET_SIZE, ALPHABET_SIZE)


def parse_bigram_file(lines) -> BigramTable:
    """`<bigram> <integer>` per line; blank lines skipped; missing bigrams are 0;
    a repeated bigram keeps its last value with a warning (ngrams.py:76-108)."""
    if isinstance(lines, str):
        lines = lines.splitlines()
    scores = np.zeros(TABLE_SIZE, dtype=np.int64)
    seen = set()
    for lineno, line in enumerate(lines, start=1):
        fields = line.split()
        if not fields:
            continue
        if len(fields) != 2:
            raise ValueError(f"line {lineno}: expected '<bigram> <score>', got {line!r}")
        bigram, value_text = fields
        if len(bigram) != 2 or any(not ("a" <= c <= "z") for c in bigram):
            raise ValueError(f"line {lineno}: bad bigram {bigram!r}")
        try:
            value = int(value_text)
        except ValueError:
            raise ValueError(f"line {lineno}: bad score {value_text!r}") from None
        if value < 0:
            raise ValueError(f"line {lineno}: negative score {value}")
        idx = bigram_index(ord(bigram[0]) - 97, ord(bigram[1]) - 97)
        if idx in seen:
            warnings.warn(f"duplicate bigram {bigram!r}; keeping the later value")
        seen.add(idx)
        scores[idx] = value
    return BigramTable(scores)


def format_bigram_file(table: BigramTable) -> str:
    """All 676 records in lexicographic order (round-trips through parse_bigram_file)."""
    rows = (f"{chr(97 + i // 26)}{chr(97 + i % 26)} {int(v)}" for i, v in enumerate(table.scores))
    return "\n".join(rows) + "\n"


def build_table_from_corpus(corpus: str) -> BigramTable:
    sym = map_text(normalize(corpus))
    if sym.size < 2:
        return BigramTable(np.zeros(TABLE_SIZE, dtype=np.int64))
    return BigramTable(np.bincount(sym[:-1] * ALPHABET_SIZE + sym[1:], minlength=TABLE_SIZE))


def build_log_table(table: BigramTable, floor: float = DEFAULT_LOG_FLOOR) -> LogBigramTable:
    """log2(count / total); zero counts get `floor`, which must lie below every
    observed bigram (ngrams.py:143-163)."""
    if floor >= 0:
        raise ValueError("floor must be negative")
    total = int(table.scores.sum())
    if total == 0:
        raise ValueError("cannot build probabilities from an all-zero table")
    seen = table.scores > 0
    logs = np.full(TABLE_SIZE, floor, dtype=np.float64)
    logs[seen] = np.log2(table.scores[seen] / total)
    if seen.any() and logs[seen].min() < floor:
        raise ValueError(
            f"floor {floor} is above the rarest observed bigram ({float(logs[seen].min()):.3f}); "
            "pass a lower floor"
        )
    return LogBigramTable(logs, floor)


def _device():
    from .engine import default_device

    return _lib.context(default_device())


def score_text_batch(texts, table: BigramTable) -> np.ndarray:
    """score_text for many texts in one GPU call."""
    flat, off = _lib.ragged(texts)
    out = np.empty(len(off) - 1, dtype=np.int64)
    ctx = _device()
    with ctx.lock:
        _lib.check(_lib.load().ccg_score_text_batch(ctx.handle, _lib.ptr(flat), _lib.ptr(off),
                                                    out.size, _lib.ptr(table.scores), _lib.ptr(out)),
                   "score_text")
    return out


def log_score_text_batch(texts, table: LogBigramTable) -> np.ndarray:
    """log_score_text for many texts in one GPU call (numpy pairwise order)."""
    flat, off = _lib.ragged(texts)
    out = np.empty(len(off) - 1, dtype=np.float64)
    ctx = _device()
    with ctx.lock:
        _lib.check(_lib.load().ccg_log_score_text_batch(ctx.handle, _lib.ptr(flat), _lib.ptr(off),
                                                        out.size, _lib.ptr(table.logs),
                                                        _lib.ptr(out)),
                   "log_score_text")
    return out


def score_text(text: MappedText, table: BigramTable) -> int:
    """Sum of table scores over adjacent letter pairs (ngrams.py:134-140), on the GPU."""
    return int(score_text_batch([text], table)[0])


def log_score_text(text: MappedText, table: LogBigramTable) -> float:
    """Sum of log2 bigram probabilities (ngrams.py:166-172), on the GPU, bit-exact."""
    return float(log_score_text_batch([text], table)[0])


# ------------------------------------------------------------------ n-gram extension
# The reference implements bigrams only (ngrams.py:21).  BASELINE.json's
# configs 3-5 ask for trigram and quadgram scoring; these classes generalise the bigram ones
# with the same conventions: index sum_j 26^(order-1-j) t_j (order 2 == bigram_index),
# non-negative integer scores summed over the text's windows, log2(count/total) with unseen
# n-grams at a floor below the rarest observed one.
def ngram_index(letters) -> int:
    idx = 0
    for x in letters:
        x = int(x)
        if not 0 <= x < ALPHABET_SIZE:
            raise ValueError(f"letter index out of range: {x}")
        idx = idx * ALPHABET_SIZE + x
    return idx


def _window_index(t: np.ndarray, order: int) -> np.ndarray:
    m = t.size - order + 1
    idx = np.zeros(max(0, m), dtype=np.int64)
    for j in range(order):
        idx = idx * ALPHABET_SIZE + t[j:j + m]
    return idx


def _check_order(order: int) -> int:
    order = int(order)
    if not 2 <= order <= 4:
        raise ValueError(f"n-gram order must be 2, 3 or 4, got {order}")
    return order


@dataclass(frozen=True)
class NgramTable:
    """26**order non-negative integer scores indexed by ngram_index (order 2 = BigramTable)."""

    order: int
    scores: np.ndarray

    def __post_init__(self):
        order = _check_order(self.order)
        arr = np.ascontiguousarray(self.scores, dtype=np.int64)
        if arr.shape != (ALPHABET_SIZE**order,):
            raise ValueError(f"expected {ALPHABET_SIZE**order} entries, got {arr.shape}")
        if arr.size and arr.min() < 0:
            raise ValueError("n-gram scores must be non-negative")
        object.__setattr__(self, "order", order)
        object.__setattr__(self, "scores", arr)


@dataclass(frozen=True)
class LogNgramTable:
    """26**order log2 n-gram probabilities; unseen n-grams sit at `floor`."""

    order: int
    logs: np.ndarray
    floor: float

    def __post_init__(self):
        order = _check_order(self.order)
        arr = np.ascontiguousarray(self.logs, dtype=np.float64)
        if arr.shape != (ALPHABET_SIZE**order,):
            raise ValueError(f"expected {ALPHABET_SIZE**order} entries, got {arr.shape}")
        if not np.isfinite(arr).all():
            raise ValueError("log scores must be finite")
        if arr.size and arr.max() > 0:
            raise ValueError("log2 probabilities cannot be positive")
        if arr.size and arr.min() < self.floor:
            raise ValueError("log table entries below the configured floor")
        object.__setattr__(self, "order", order)
        object.__setattr__(self, "logs", arr)


def as_ngram_table(table) -> NgramTable:
    """BigramTable -> NgramTable(2, ...); NgramTable passes through."""
    if isinstance(table, NgramTable):
        return table
    if isinstance(table, BigramTable):
        return NgramTable(2, table.scores)
    raise TypeError(f"not a score table: {type(table).__name__}")


def as_log_ngram_table(table) -> LogNgramTable:
    if isinstance(table, LogNgramTable):
        return table
    if isinstance(table, LogBigramTable):
        return LogNgramTable(2, table.logs, table.floor)
    raise TypeError(f"not a log table: {type(table).__name__}")


def build_ngram_table_from_corpus(corpus: str, order: int) -> NgramTable:
    """Count the normalized corpus's windows of `order` letters (build_table_from_corpus,
    ngrams.py:124-131, generalised)."""
    order = _check_order(order)
    sym = map_text(normalize(corpus))
    counts = np.zeros(ALPHABET_SIZE**order, dtype=np.int64)
    if sym.size >= order:
        counts = np.bincount(_window_index(sym, order), minlength=ALPHABET_SIZE**order)
    return NgramTable(order, counts.astype(np.int64))


def build_log_ngram_table(table: NgramTable, floor: float = DEFAULT_LOG_FLOOR) -> LogNgramTable:
    """log2(count / total); zero counts get `floor` (ngrams.py:143-163 generalised)."""
    table = as_ngram_table(table)
    if floor >= 0:
        raise ValueError("floor must be negative")
    total = int(table.scores.sum())
    if total == 0:
        raise ValueError("cannot build probabilities from an all-zero table")
    seen = table.scores > 0
    logs = np.full(table.scores.size, floor, dtype=np.float64)
    logs[seen] = np.log2(table.scores[seen] / total)
    if seen.any() and logs[seen].min() < floor:
        raise ValueError(
            f"floor {floor} is above the rarest observed n-gram ({float(logs[seen].min()):.3f}); "
            "pass a lower floor"
        )
    return LogNgramTable(table.order, logs, floor)


def quantize_log_table(table, max_value: int = 65535) -> NgramTable:
    """Integer fitness table for the MAS climb: the affine map [floor, 0] -> [0, max_value]
    of the log2 probabilities, rounded.  For a fixed text length the integer score is an
    increasing affine function of the (rounded) log-probability sum, so the climb ranks
    candidates as the log score does; entries fit the kernels' uint16 tables."""
    t = as_log_ngram_table(table)
    if not 1 <= int(max_value) <= 65535:
        raise ValueError("max_value must lie in 1..65535")
    q = np.rint((t.logs - t.floor) / (-t.floor) * int(max_value)).astype(np.int64)
    return NgramTable(t.order, np.clip(q, 0, int(max_value)))


@dataclass(frozen=True)
class QuantizedSctTable:
    """Integer fitness of the opt-in fast SCT mode (engine.sct_fast_climb): table[i] =
    round(logs[i] * 2**shift), int32, <= 0.  Integer sums are exact and associative, which is
    what lets the climb re-score only the windows a candidate changes; the float64 parity
    path (sct.py:158-160) cannot be updated incrementally and stay bit-exact."""

    order: int
    table: np.ndarray
    shift: int


def quantize_sct_table(table, text_len: int = 4096, max_shift: int = 16) -> QuantizedSctTable:
    """Quantise a log table (LogBigramTable / LogNgramTable) for the fast SCT mode with the
    largest shift <= max_shift whose fitness cannot overflow int32 for texts of up to
    `text_len` letters: (text_len - order + 1) * max|entry| < 2**31."""
    t = as_log_ngram_table(table)
    windows = max(1, int(text_len) - t.order + 1)
    worst = float(np.max(np.abs(t.logs))) if t.logs.size else 0.0
    shift = int(max_shift)
    while shift > 0 and windows * np.rint(worst * 2.0**shift) >= 2**31:
        shift -= 1
    if windows * np.rint(worst * 2.0**shift) >= 2**31:
        raise ValueError("log table too large to quantise for this text length")
    q = np.rint(t.logs * 2.0**shift).astype(np.int64)
    return QuantizedSctTable(t.order, q.astype(np.int32), shift)


def ngram_score_text_batch(texts, table) -> np.ndarray:
    """Integer n-gram fitness of many texts in one GPU call."""
    t = as_ngram_table(table)
    from .engine import ngram_score_batch

    return ngram_score_batch(texts, t.order, t.scores)


def ngram_score_text(text: MappedText, table) -> int:
    """Sum of table entries over the text's windows (score_text generalised), on the GPU."""
    return int(ngram_score_text_batch([text], table)[0])


def ngram_log_score_text_batch(texts, table) -> np.ndarray:
    """Log-probability fitness of many texts (log_score_text generalised), bit-exact numpy
    pairwise order, in one GPU call."""
    t = as_log_ngram_table(table)
    from .engine import ngram_log_score_batch

    return ngram_log_score_batch(texts, t.order, t.logs)


def ngram_log_score_text(text: MappedText, table) -> float:
    return float(ngram_log_score_text_batch([text], table)[0])


def parse_ngram_file(lines, order: int) -> NgramTable:
    """`<ngram> <integer>` per line (parse_bigram_file, ngrams.py:76-108, generalised to
    windows of `order` letters): blank lines skipped, missing n-grams are 0, a repeated
    n-gram keeps its last value with a warning."""
    order = _check_order(order)
    if isinstance(lines, str):
        lines = lines.splitlines()
    scores = np.zeros(ALPHABET_SIZE**order, dtype=np.int64)
    seen = set()
    for lineno, line in enumerate(lines, start=1):
        fields = line.split()
        if not fields:
            continue
        if len(fields) != 2:
            raise ValueError(f"line {lineno}: expected '<ngram> <score>', got {line!r}")
        gram, value_text = fields
        if len(gram) != order or any(not ("a" <= ch <= "z") for ch in gram):
            raise ValueError(f"line {lineno}: bad {order}-gram {gram!r}")
        try:
            value = int(value_text)
        except ValueError:
            raise ValueError(f"line {lineno}: bad score {value_text!r}") from None
        if value < 0:
            raise ValueError(f"line {lineno}: negative score {value}")
        idx = ngram_index(ord(ch) - 97 for ch in gram)
        if idx in seen:
            warnings.warn(f"duplicate {order}-gram {gram!r}; keeping the later value")
        seen.add(idx)
        scores[idx] = value
    return NgramTable(order, scores)


def format_ngram_file(table, nonzero_only: bool = False) -> str:
    """All 26**order records in lexicographic order (format_bigram_file generalised; at
    order 2 the output is identical).  nonzero_only drops zero entries, which
    parse_ngram_file restores as 0."""
    t = as_ngram_table(table)
    out = []
    for i, v in enumerate(t.scores):
        if nonzero_only and not v:
            continue
        letters, x = [], i
        for _ in range(t.order):
            letters.append(chr(97 + x % ALPHABET_SIZE))
            x //= ALPHABET_SIZE
        out.append(f"{''.join(reversed(letters))} {int(v)}")
    return "\n".join(out) + "\n"
