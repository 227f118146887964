#!/usr/bin/env python
"""How much of an SCT candidate the fast mode must re-read: for random keys
and the reference's operators (sct.py:82-135, applied by the oracle, oracle/cc_oracle.c
cco_apply_operator) with the default mix (p1=33, p2=66, hops 3/3), count the order-gram
windows that touch a column whose segment offset moved, as a fraction of all windows.
Prints one JSON line per (order, k) and the C3 average (k = 5..20, n = 400)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402


def starts(key, n):
    k = key.size
    base, rem = divmod(n, k)
    lens = np.where(np.arange(k) < rem, base + 1, base)
    out = np.zeros(k, np.int64)
    s = 0
    for p in range(k):
        out[key[p]] = s
        s += lens[key[p]]
    return out


def windows_touched(key, cand, n, order):
    k = key.size
    moved = np.nonzero(starts(key, n) != starts(cand, n))[0]
    dirty = {(c - i) % k for c in moved for i in range(order)}
    items = sum(len(range(w, n - order + 1, k)) for w in dirty)
    return items, n - order + 1


def main(trials=2000, n=400):
    rng = np.random.default_rng(5)
    out = []
    for order in (2, 3):
        tot_items = tot_all = 0
        for k in range(5, 21):
            items = alls = 0
            for t in range(trials):
                key = rng.permutation(k)
                u = int(rng.integers(0, 100))
                op = 1 if u < 33 else 2 if u < 66 else 3
                cand = O.apply_operator(op, key, 3, 1000 * k + t, order, 1)[0]
                a, b = windows_touched(key, cand, n, order)
                items += a
                alls += b
            out.append({"order": order, "k": k, "n": n, "windows_reread_per_eval": items / trials,
                        "of": alls / trials, "fraction": items / alls})
            tot_items += items
            tot_all += alls
        out.append({"order": order, "k": "5..20 (C3)", "n": n, "fraction": tot_items / tot_all})
    for line in out:
        print(json.dumps(line))


if __name__ == "__main__":
    main()
