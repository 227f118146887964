"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the dev container (the reference is only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything written here is an output of the reference `cipherclimb` package
(/root/reference/pkg/src/cipherclimb, numpy 2.3.5) or of numpy's own generators,
so the fixtures pin the oracle (oracle/cc_oracle.c) and the CUDA engine to the
reference's exact behaviour on the GPU box, where /root/reference does not exist.
Inputs that numpy regenerates cheaply (default_rng-seeded texts) are NOT stored:
the tests rebuild them with the same recipe and only the reference outputs are kept.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

import cipherclimb as cc
from cipherclimb.rng import KEYGEN_STREAM, worker_stream_index

OUT = Path(__file__).resolve().parent
DATA = Path("/root/reference/pkg/data")

t0 = time.time()


def log(msg):
    print(f"[{time.time() - t0:7.1f}s] {msg}", flush=True)


# ----------------------------------------------------------------- data
corpus = (DATA / "corpus.txt").read_text()
table = cc.build_table_from_corpus(corpus)
shipped = cc.parse_bigram_file((DATA / "english_bigrams.txt").read_text())
assert np.array_equal(table.scores, shipped.scores)
logs = cc.build_log_table(table)
plain_mas_full = cc.map_text(cc.normalize((DATA / "sample_plain_mas.txt").read_text()))
plain_sct_full = cc.map_text(cc.normalize((DATA / "sample_plain_sct.txt").read_text()))
corpus_mapped = cc.map_text(cc.normalize(corpus))
np.savez_compressed(
    OUT / "data.npz",
    english_scores=table.scores,
    english_logs=logs.logs,
    english_floor=np.float64(logs.floor),
    plain_mas=plain_mas_full.astype(np.uint8),
    plain_sct=plain_sct_full.astype(np.uint8),
    corpus=corpus_mapped.astype(np.uint8),
)
log(f"data: corpus {corpus_mapped.size} letters, mas {plain_mas_full.size}, sct {plain_sct_full.size}")

# ----------------------------------------------------------------- rng
RNG_KEYS = [
    (0, 0), (7, 3), (12345, (5 << 32) | 17), (2**63 - 1, 2**32 - 1), (-1, 0),
    (2**64 - 1, 2**64 - 1), (42, KEYGEN_STREAM), (7000, worker_stream_index(19, 63)),
]
def _draws(s, w, n):
    st = cc.WorkerRng(s, w)
    return [st.next_uniform() for _ in range(n)]


uniforms = np.array([_draws(s, w, 300) for s, w in RNG_KEYS])
BOUNDS = [1, 2, 3, 7, 10, 26, 99, 100, 1000]
int_seq = {}
for b in BOUNDS:
    st = cc.WorkerRng(11, b)
    int_seq[b] = np.array([st.next_int_below(b) for _ in range(2000)])
pairs = {}
for b in (2, 3, 10, 26):
    st = cc.WorkerRng(17, b)
    pairs[b] = np.array([st.next_distinct_pair(b) for _ in range(2000)])
perms = {n: cc.WorkerRng(19, n).permutation(n) for n in (1, 2, 3, 5, 10, 15, 20, 26, 40, 64)}
np.savez_compressed(
    OUT / "rng.npz",
    keys_seed=np.array([s % 2**64 for s, _ in RNG_KEYS], dtype=np.uint64),
    keys_stream=np.array([w % 2**64 for _, w in RNG_KEYS], dtype=np.uint64),
    uniforms=uniforms,
    bounds=np.array(BOUNDS),
    **{f"int_seq_{b}": v for b, v in int_seq.items()},
    **{f"pairs_{b}": v for b, v in pairs.items()},
    **{f"perm_{n}": v for n, v in perms.items()},
)
log("rng")

# ----------------------------------------------------------------- scoring
# score_text / log_score_text on texts rebuilt by tests: default_rng(900 + i), length L_i
score_lengths = list(range(0, 140)) + [199, 255, 256, 257, 300, 399, 400, 471, 500, 595, 596,
                                      1000, 1025, 2048, 4097]
rnd_table = cc.BigramTable(np.random.default_rng(901).integers(0, 900, 676))
int_scores, eng_scores, log_scores = [], [], []
for i, L in enumerate(score_lengths):
    t = np.random.default_rng(900 + i).integers(0, 26, L)
    int_scores.append(cc.score_text(t, rnd_table))
    eng_scores.append(cc.score_text(t, table))
    log_scores.append(cc.log_score_text(t, logs))
np.savez_compressed(
    OUT / "scoring.npz",
    lengths=np.array(score_lengths),
    rnd_table=rnd_table.scores,
    int_scores=np.array(int_scores),
    eng_scores=np.array(eng_scores),
    log_scores=np.array(log_scores),
)
log("scoring")

# acceptance #05 recipe (tests/test_acceptance.py:113-124): 10,000 swaps, seed 501
rng = np.random.default_rng(501)
t05 = cc.BigramTable(rng.integers(0, 900, 676))
deltas = []
for _ in range(10_000):
    text = rng.integers(0, 26, int(rng.integers(2, 220)))
    a, b = (int(v) for v in rng.choice(26, size=2, replace=False))
    deltas.append(cc.text_swap_delta(text, a, b, t05))
np.savez_compressed(OUT / "mas_delta.npz", deltas=np.array(deltas))
log("mas_delta")

# ----------------------------------------------------------------- SCT primitives
gm_cases = []
gm_maps = []
for k in range(1, 41):
    for n in (k, k + 1, 2 * k + 3, 5 * k - 1 if k > 1 else 4):
        key = cc.WorkerRng(k * 1000 + n, 0).permutation(k)
        gm_cases.append((k, n))
        gm_maps.append(cc.transposition_gather_map(key, n))
np.savez_compressed(
    OUT / "sct_gather.npz",
    cases=np.array(gm_cases),
    maps=np.concatenate(gm_maps),
)
ops = {}
for k in (2, 3, 5, 8, 13, 25, 40):
    key = cc.WorkerRng(46, k).permutation(k)
    ops[f"key{k}"] = key
    for op, fn in ((1, lambda kk, st: cc.apply_element_swaps(kk, st, 3)),
                   (2, lambda kk, st: cc.apply_block_swaps(kk, st, 3)),
                   (3, lambda kk, st: cc.apply_block_shift(kk, st))):
        st = cc.WorkerRng(46, 100 * k + op)  # one fresh stream per operator
        ops[f"k{k}_op{op}"] = np.array([fn(key, st) for _ in range(200)])
np.savez_compressed(OUT / "sct_ops.npz", **ops)
log("sct primitives")

# ----------------------------------------------------------------- MAS workers
# Case i: ciphertext = mas_encrypt(window of plain_mas_full / corpus, key_i), various tables.
mas_cases = []  # (source, offset, length, key_seed, table_id, climbings, seed, stream)
specs = [
    # length, climbings, table (0 english, 1 random 0..899, 2 random 0..60000), source
    (2, 50, 0, "mas"), (3, 200, 1, "mas"), (26, 1000, 0, "mas"), (60, 3000, 0, "corpus"),
    (100, 5000, 0, "corpus"), (150, 1500, 1, "corpus"), (300, 10000, 0, "mas"),
    (300, 4000, 2, "corpus"), (471, 10000, 0, "mas"), (500, 10000, 0, "corpus"),
    (637, 2000, 1, "mas"), (1500, 3000, 0, "corpus"),
]
tables = {0: table, 1: t05, 2: cc.BigramTable(np.random.default_rng(77).integers(0, 60000, 676))}
mw = {"lengths": [], "offsets_src": [], "src": [], "key_seed": [], "table_id": [], "climbings": [],
      "seed": [], "stream": [], "score": [], "text": []}
for i, (L, climb, tid, src) in enumerate(specs):
    source = plain_mas_full if src == "mas" else corpus_mapped
    off = int(np.random.default_rng(i).integers(0, max(1, source.size - L)))
    plain = source[off:off + L]
    key = cc.WorkerRng(3000 + i, KEYGEN_STREAM).permutation(26)
    cipher = cc.mas_encrypt(plain, key)
    if np.unique(cipher).size < 2:
        continue
    for j, (seed, stream) in enumerate([(5 + i, worker_stream_index(0, j)) for j in range(2)] +
                                       [(2**63 + i, worker_stream_index(3, 77))]):
        text, score = cc.stochastic_worker(cipher, tables[tid], climb, cc.WorkerRng(seed, stream))
        mw["lengths"].append(L); mw["offsets_src"].append(off); mw["src"].append(src == "corpus")
        mw["key_seed"].append(3000 + i); mw["table_id"].append(tid); mw["climbings"].append(climb)
        mw["seed"].append(seed); mw["stream"].append(stream); mw["score"].append(score)
        mw["text"].append(text.astype(np.uint8))
np.savez_compressed(
    OUT / "mas_workers.npz",
    table1=t05.scores, table2=tables[2].scores,
    lengths=np.array(mw["lengths"]), offsets_src=np.array(mw["offsets_src"]),
    src_corpus=np.array(mw["src"]), key_seed=np.array(mw["key_seed"]),
    table_id=np.array(mw["table_id"]), climbings=np.array(mw["climbings"]),
    seed=np.array(mw["seed"], dtype=np.uint64), stream=np.array(mw["stream"], dtype=np.uint64),
    score=np.array(mw["score"]), text=np.concatenate(mw["text"]),
)
log(f"mas workers: {len(mw['score'])}")

# solve_stochastic on acceptance #07 experiment 0 inputs (471 letters), restarts 0 and 1
plain471 = plain_mas_full[:471]
key7 = cc.WorkerRng(700, KEYGEN_STREAM).permutation(26)
cipher7 = cc.mas_encrypt(plain471, key7)
cfg7 = cc.MasSolverConfig(workers=64, climbings=10_000, restarts=20, global_seed=7000)
solves = []
for r in range(2):
    res = cc.solve_stochastic(cipher7, table, cfg7, jobs=8, restart=r)
    solves.append(res)
np.savez_compressed(
    OUT / "mas_solve.npz",
    cipher=cipher7.astype(np.uint8),
    per_worker=np.array([s.per_worker_scores for s in solves]),
    best_text=np.array([s.best_text for s in solves]).astype(np.uint8),
    best_score=np.array([s.best_score for s in solves]),
)
log("mas solve_stochastic x2")

# ----------------------------------------------------------------- SCT workers
sct_specs = [
    # (k, n, climbings, table: 0 english log, 1 tiny random log)
    (2, 20, 100, 1), (3, 60, 500, 1), (4, 80, 2000, 0), (5, 400, 3000, 0), (6, 60, 1000, 1),
    (7, 70, 800, 1), (10, 400, 5000, 0), (10, 596, 15000, 0), (13, 300, 2000, 0),
    (15, 596, 6000, 0), (20, 400, 4000, 0), (24, 500, 2000, 0), (32, 640, 1500, 0),
    (40, 800, 1000, 0), (9, 8, 0, 1),
]
tiny = cc.build_log_table(cc.BigramTable(np.random.default_rng(40).integers(1, 300, 676)))
ltabs = {0: logs, 1: tiny}
sw = {k: [] for k in ("k", "n", "climbings", "table_id", "key_seed", "seed", "stream", "score",
                      "key", "cipher")}
for i, (k, n, climb, tid) in enumerate(sct_specs):
    if n < k:
        continue
    src = np.concatenate([plain_sct_full, plain_mas_full])
    off = int(np.random.default_rng(100 + i).integers(0, src.size - n))
    plain = src[off:off + n]
    key = cc.WorkerRng(4000 + i, KEYGEN_STREAM).permutation(k)
    cipher = cc.sct_encrypt(plain, key)
    cfg = cc.SctSolverConfig(key_length=k, climbings=climb, workers=1)
    for seed, stream in [(8000 + i, worker_stream_index(0, 0)), (8000 + i, worker_stream_index(1, 5))]:
        kk, score = cc.sct_worker(cipher, ltabs[tid], cfg, cc.WorkerRng(seed, stream))
        sw["k"].append(k); sw["n"].append(n); sw["climbings"].append(climb); sw["table_id"].append(tid)
        sw["key_seed"].append(4000 + i); sw["seed"].append(seed); sw["stream"].append(stream)
        sw["score"].append(score); sw["key"].append(kk); sw["cipher"].append(cipher.astype(np.uint8))
    log(f"sct worker k={k} n={n}")
np.savez_compressed(
    OUT / "sct_workers.npz",
    tiny_logs=tiny.logs, tiny_floor=np.float64(tiny.floor),
    k=np.array(sw["k"]), n=np.array(sw["n"]), climbings=np.array(sw["climbings"]),
    table_id=np.array(sw["table_id"]), key_seed=np.array(sw["key_seed"]),
    seed=np.array(sw["seed"], dtype=np.uint64), stream=np.array(sw["stream"], dtype=np.uint64),
    score=np.array(sw["score"]), key=np.concatenate(sw["key"]), cipher=np.concatenate(sw["cipher"]),
)

# solve_sct: acceptance #08 shape, k=10 experiment 0, restart 0 only (64 workers x 15k)
plain596 = plain_sct_full[:596]
key8 = cc.WorkerRng(800, KEYGEN_STREAM).permutation(10)
cipher8 = cc.sct_encrypt(plain596, key8)
cfg8 = cc.SctSolverConfig(key_length=10, workers=64, climbings=15_000, restarts=1, global_seed=8000)
best8, _ = cc.solve_sct(cipher8, logs, cfg8, jobs=8)
np.savez_compressed(
    OUT / "sct_solve.npz",
    cipher=cipher8.astype(np.uint8),
    per_worker=np.array(best8.per_worker_scores),
    best_key=best8.best_key,
    best_text=best8.best_text.astype(np.uint8),
    best_score=np.float64(best8.best_score),
    recovered=np.array(np.array_equal(best8.best_text, plain596)),
)
log("sct solve")
print("done", file=sys.stderr)
