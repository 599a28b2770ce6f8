"""Pure-Python exact / brute-force checks for tiny inputs -- TEST INFRASTRUCTURE ONLY.

Used only by tests/ to pin oracle/ref.py:
* ``topk_bruteforce``: the kept chunk set as the lexicographically smallest
  maximum-sum K-subset, with sums compared exactly as Fractions ("select
  the Top-K blocks"; tie rule Z10).  This is a definition independent of any
  sort order, so it pins ``ref.select_chunks``.
* ``pooled_exact``: the shrinking-window mean with Fractions (Z6).
"""
from __future__ import annotations

import itertools
from fractions import Fraction


def topk_bruteforce(scores, K):
    """All C(n, K) subsets; maximise the exact sum, then the lexicographically
    smallest sorted index tuple."""
    fr = [Fraction(float(s)) for s in scores]
    best_sum, best = None, None
    for sub in itertools.combinations(range(len(fr)), K):   # generated in lexicographic order
        s = sum(fr[i] for i in sub)
        if best_sum is None or s > best_sum:                # strict: the first (smallest) tuple wins ties
            best_sum, best = s, sub
    return list(best)


def pooled_exact(values, pool_k):
    fr = [Fraction(float(v)) for v in values]
    n, w = len(fr), (pool_k - 1) // 2
    out = []
    for i in range(n):
        win = fr[max(0, i - w):min(n, i + w + 1)]
        out.append(sum(win) / len(win))
    return out
