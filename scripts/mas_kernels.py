#!/usr/bin/env python
"""Time the MAS kernel variants on the bench workload (C2, device-resident inputs):
python scripts/mas_kernels.py [--ciphers N] [kernels...]"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import torch  # noqa: E402
from paper_2103_13937_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ciphers", type=int, default=10_000)
ap.add_argument("kernels", nargs="*", default=["dform", "dtable", "tform"])
a = ap.parse_args()
ctx = _lib.context(0)
L = _lib.load()
plains, ciphers, scores, lengths = bench.make_workload(a.ciphers, 0)
W, K = 64, 10_000
keys = bench.worker_keys(len(ciphers), W, 0)
flat, off = _lib.ragged(ciphers)
cof = np.repeat(np.arange(len(ciphers), dtype=np.int32), W)
n = len(ciphers) * W


def dev(arr):
    p = ctx.dev_alloc(max(1, arr.nbytes))
    ctx.h2d(p, np.ascontiguousarray(arr))
    return p


args = _lib.MasClimbArgs()
args.ciphers, args.offsets, args.n_ciphers = dev(flat), dev(off), len(ciphers)
args.cipher_of, args.keys, args.skips = dev(cof), dev(keys), None
args.n_workers, args.climbings, args.table = n, K, dev(scores)
args.scores = ctx.dev_alloc(n * 8)
args.max_len, args.table_max = int(lengths.max()), int(scores.max())
stream = torch.cuda.ExternalStream(ctx.stream(), device="cuda:0")
ref = None
for kern in a.kernels:
    args.flags = _lib.KERNEL_FLAGS[kern]
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
        _lib.check(L.ccg_mas_climb_dev(ctx.handle, args), kern)
        with torch.cuda.stream(stream):
            e1.record(stream)
        ctx.synchronize()
        ms = e0.elapsed_time(e1)
    sc = np.empty(n, dtype=np.int64)
    ctx.d2h(sc, args.scores)
    ctx.synchronize()
    same = ref is None or np.array_equal(sc, ref)
    ref = sc if ref is None else ref
    print(f"{kern:8s} {n * K / ms / 1e6:.4g} evals/s  ({ms:.2f} ms)  scores match: {same}", flush=True)
