"""Oracle finalize: exact integer moments -> mean, variance, 90% CI half-width.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

SPEC S:398-405 (StatPoint), S:418-427 (worked values), S:440-445 (z = 1.6449,
90% two-sided normal interval); PAPER Fig. 1 caption ("variance
(90% confidence)").  From count n, S1 = sum v, S2 = sum v^2 (Python ints, exact):
    mean = S1 / n
    var  = (n*S2 - S1^2) / (n (n-1))     unbiased; 0 when n == 1
    ci90 = 1.6449 * sqrt(var / n)
mean and var are formed as exact rationals and rounded once to fp64.
"""
from __future__ import annotations

import math
from fractions import Fraction

Z90 = 1.6449


def finalize_cell(n, s1, s2):
    n, s1, s2 = int(n), int(s1), int(s2)
    if n <= 0:
        return float("nan"), float("nan"), float("nan")
    mean = float(Fraction(s1, n))
    if n == 1:
        return mean, 0.0, 0.0
    var = float(Fraction(n * s2 - s1 * s1, n * (n - 1)))
    ci = Z90 * math.sqrt(var / n)
    return mean, var, ci


def sumsq_int(sq):
    """(lo, hi) uint64 pair -> Python int."""
    return int(sq[0]) | (int(sq[1]) << 64)


def finalize(count, s1, sumsq_pairs):
    """Elementwise over flat arrays; returns three lists of floats."""
    means, vars_, cis = [], [], []
    cnt = list(count.reshape(-1))
    sm = list(s1.reshape(-1))
    sq = sumsq_pairs.reshape(-1, 2)
    for i in range(len(cnt)):
        m, v, c = finalize_cell(cnt[i], sm[i], sumsq_int(sq[i]))
        means.append(m)
        vars_.append(v)
        cis.append(c)
    return means, vars_, cis
