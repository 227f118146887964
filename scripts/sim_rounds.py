#!/usr/bin/env python
"""Tries covered per D-form round (ccg_mas_dform.cu) over a uniform letter stream: the round-1
two-segment rounds (up to the second redraw) vs the round-2 three-segment rounds (the pairs
realign after a second redraw, one lane further on; rounds cap at 31 pairs then).
A redraw is a pair whose two letters are equal (rng.py:85-86)."""
import numpy as np


def tries_per_round(seg3: bool, n_draws: int = 60_000, seed: int = 1) -> float:
    d = np.random.default_rng(seed).integers(0, 26, n_draws + 300)
    o = tries = rounds = 0
    while o < n_draws:
        c = [(d[o + 2 * j], d[o + 2 * j + 1], d[o + 2 * j + 2]) for j in range(33)]
        r0 = next((j for j in range(32) if c[j][0] == c[j][1]), 32)
        R, r1, seq = 32, 32, False
        if r0 < 32:
            if c[r0][2] == c[r0][0]:
                R, seq = r0, True
            else:
                rb = next((j for j in range(r0 + 1, 32) if c[j][1] == c[j][2]), 32)
                if rb < 32:
                    if not seg3 or rb == 31 or c[rb + 1][1] == c[rb][1]:
                        R = rb
                    else:
                        r1 = rb
                        R = next((j for j in range(r1 + 1, 31) if c[j + 1][0] == c[j + 1][1]), 31)
        o += 2 * R + (R > r0) + (R > r1)
        tries += R
        rounds += 1
        if seq:  # one try through the sequential pair path
            a, b = d[o], d[o + 1]
            o += 2
            while b == a:
                b = d[o]
                o += 1
            tries += 1
    return tries / rounds


if __name__ == "__main__":
    print(f"two segments: {tries_per_round(False):.1f} tries per round; "
          f"three segments: {tries_per_round(True):.1f}")
