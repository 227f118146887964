"""Multi-process restart sharding (paper_2103_13937_b200.parallel) at world_size 2 over gloo
on CPU.  Each rank's GPU climb is replaced by the oracle, so the host-side sharding,
gather and lexicographic best-over-ranks logic is exercised against reference-exact
per-worker results; the result must equal the single-process solve."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def oracle_climb(ciphers, cipher_of, keys, table, climbings, group_size=0, **_):
    """engine.mas_climb stand-in: the oracle on raw Philox keys."""
    from oracle import oracle as O
    from paper_2103_13937_b200.engine import ClimbResult

    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, 2)
    flat, off = O.ragged(ciphers)
    scores, maps = [], []
    for c, (k0, k1) in zip(cipher_of, keys):
        t = flat[off[c]:off[c + 1]]
        out_text = np.empty(t.size, np.int64)
        out_map = np.empty(26, np.int64)
        s = O.lib().cco_stochastic_worker(O._p(t), t.size, O._p(np.asarray(table, np.int64)),
                                          int(climbings), int(k0), int(k1), 0, O._p(out_text),
                                          O._p(out_map), None)
        scores.append(s)
        maps.append(out_map)
    scores = np.array(scores, dtype=np.int64)
    gb = None
    if group_size:
        gb = np.array([int(np.argmax(scores[i:i + group_size]))
                       for i in range(0, scores.size, group_size)], dtype=np.int64)
    return ClimbResult(scores=scores, keys=np.array(maps), group_best=gb, draws_used=None,
                       last_accept=None, tries_done=None, launches=0)


def oracle_sct_climb(ciphers, cipher_of, keys, logs, key_length, climbings, p1=33, p2=66,
                     op1_hop=3, op2_hop=3, group_size=0, order=2, **_):
    """engine.sct_climb stand-in: the oracle on raw Philox keys."""
    from oracle import oracle as O
    from paper_2103_13937_b200.engine import ClimbResult

    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, 2)
    flat, off = O.ragged(ciphers)
    cfg = O._cfgv(key_length, climbings, p1, p2, op1_hop, op2_hop, order)
    lg = np.ascontiguousarray(logs, dtype=np.float64)
    scores, outk = [], []
    for c, (k0, k1) in zip(cipher_of, keys):
        t = flat[off[c]:off[c + 1]]
        kk = np.empty(key_length, np.int64)
        s = O.lib().cco_sct_worker(O._p(t), t.size, O._p(lg), O._p(cfg), int(k0), int(k1), 0,
                                   O._p(kk), None)
        scores.append(s)
        outk.append(kk)
    scores = np.array(scores, dtype=np.float64)
    gb = np.array([int(np.argmax(scores[i:i + group_size]))
                   for i in range(0, scores.size, group_size)], dtype=np.int64)
    return ClimbResult(scores=scores, keys=np.array(outk), group_best=gb, draws_used=None,
                       last_accept=None, tries_done=None, launches=0)


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2103_13937_b200 as cc
        from paper_2103_13937_b200 import parallel

        from test_parallel_gloo import oracle_climb

        rng = np.random.default_rng(4)
        table = cc.BigramTable(rng.integers(0, 900, 676))
        cipher = rng.integers(0, 26, 200)
        out = {}
        for W in (6, 1, 5):
            cfg = cc.MasSolverConfig(workers=W, climbings=700, global_seed=99)
            res = parallel.solve_stochastic_sharded(cipher, table, cfg, restart=1,
                                                    climb=oracle_climb)
            out[W] = (res.best_score, res.per_worker_scores, res.best_text.tolist())
        logs = cc.build_log_table(cc.BigramTable(rng.integers(1, 500, 676)))
        sc = rng.integers(0, 26, 150)
        for W in (5, 2):
            scfg = cc.SctSolverConfig(key_length=6, workers=W, climbings=300, global_seed=17)
            res = parallel.solve_sct_sharded(sc, logs, scfg, restart=2, climb=oracle_sct_climb)
            out[("sct", W)] = (res.best_score, res.per_worker_scores, res.best_key.tolist(),
                               res.best_text.tolist())
        # tie-break: equal scores on both ranks -> lowest global index wins
        s, i, p = parallel.best_over_ranks(10, 7 - rank, np.full(3, rank))
        out["tie"] = (s, i, p.tolist())
        s, i, p = parallel.best_over_ranks(2.5 + rank, rank, np.full(2, rank))
        out["float"] = (s, i, p.tolist())
        out["gather"] = parallel.all_gather_array(np.arange(10 * rank, 13 * rank, dtype=np.int64)).tolist()
        out["slice"] = parallel.rank_slice(10)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_solve_matches_single_process():
    import paper_2103_13937_b200 as cc
    from paper_2103_13937_b200.rng import philox_keys, worker_stream_index

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    rng = np.random.default_rng(4)
    table = cc.BigramTable(rng.integers(0, 900, 676))
    cipher = rng.integers(0, 26, 200)
    for W in (6, 1, 5):
        keys = philox_keys([99], [worker_stream_index(1, w) for w in range(W)])
        ref = oracle_climb([cipher], np.zeros(W, np.int32), keys, table.scores, 700, group_size=W)
        best = int(ref.group_best[0])
        want = (int(ref.scores[best]), ref.scores.tolist(), ref.keys[best][cipher].tolist())
        assert results[0][W] == want and results[1][W] == want, W
    logs = cc.build_log_table(cc.BigramTable(rng.integers(1, 500, 676)))
    sc = rng.integers(0, 26, 150)
    for W in (5, 2):
        keys = philox_keys([17], [worker_stream_index(2, w) for w in range(W)])
        ref = oracle_sct_climb([sc], np.zeros(W, np.int32), keys, logs.logs, 6, 300, group_size=W)
        best = int(ref.group_best[0])
        want = (float(ref.scores[best]), ref.scores.tolist(), ref.keys[best].tolist(),
                cc.sct_decrypt(sc, ref.keys[best]).tolist())
        assert results[0][("sct", W)] == want and results[1][("sct", W)] == want, W
    assert results[0]["tie"] == results[1]["tie"] == (10, 6, [1, 1, 1])
    assert results[0]["float"] == results[1]["float"] == (3.5, 1, [1, 1])
    assert results[0]["gather"] == results[1]["gather"] == [10, 11, 12]
    assert results[0]["slice"] == (0, 5) and results[1]["slice"] == (5, 10)
