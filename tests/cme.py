"""Chemical master equation by brute force on tiny state spaces (test helper).

Independent of oracle/ and of the CUDA path: the reachable states of a
single-compartment mass-action model are enumerated by breadth-first search
from x0, the generator Q (Q[s, s'] = sum of propensities of reactions taking
s to s'; Q[s, s] = -sum) is built from the textbook mass-action propensity
k * prod C(x_i, m_i) (Gillespie 1977), and
p(t) = p(0) expm(Q t) with scipy.linalg.expm.
"""
import math

import numpy as np
from scipy.linalg import expm


def _reactions(desc):
    out = []
    S = desc["n_species"]
    for r in desc["rules"]:
        re = [0] * S
        pr = [0] * S
        for (_, s, m) in r["reactants"]:
            re[s] += m
        for (_, s, m) in r["products"]:
            pr[s] += m
        out.append((float(r["rate"]), re, [p - q for p, q in zip(pr, re)]))
    return out


def solve(desc, times, max_states=5000, cap=10**6):
    rx = _reactions(desc)
    x0 = tuple(desc["init"])
    index = {x0: 0}
    states = [x0]
    edges = []
    i = 0
    while i < len(states):
        x = states[i]
        for (k, re, nu) in rx:
            h = 1
            for xs, m in zip(x, re):
                h *= math.comb(xs, m)
            if h == 0:
                continue
            y = tuple(a + b for a, b in zip(x, nu))
            if max(y) > cap:
                raise ValueError("state space not finite under cap")
            if y not in index:
                index[y] = len(states)
                states.append(y)
                if len(states) > max_states:
                    raise ValueError("state space too large")
            edges.append((i, index[y], k * h))
        i += 1
    n = len(states)
    Q = np.zeros((n, n))
    for a, b, rate in edges:
        Q[a, b] += rate
        Q[a, a] -= rate
    p0 = np.zeros(n)
    p0[0] = 1.0
    return states, [p0 @ expm(Q * t) for t in times]


def chi2_pvalue(observed, expected_p, n, min_expected=5.0):
    """Pearson chi^2 with pooling of small-expectation bins into one."""
    from scipy.stats import chi2
    exp = np.asarray(expected_p) * n
    obs = np.asarray(observed, dtype=float)
    big = exp >= min_expected
    o = list(obs[big]) + [obs[~big].sum()]
    e = list(exp[big]) + [exp[~big].sum()]
    if e[-1] < 1e-12:
        o, e = o[:-1], e[:-1]
    o, e = np.asarray(o), np.asarray(e)
    stat = ((o - e) ** 2 / e).sum()
    df = max(len(e) - 1, 1)
    return float(chi2.sf(stat, df))
