"""Pins for the oracle's flattening, combination counting and selection.

- P:193-196 (paper's only worked example): rule l: a b X -> c X on a a b b
  gives 4 combinations and rate 4k.
- SPEC S:134-136: binomial / match_populations examples.
- SPEC S:212-214: selection examples.
- Brute force: combination counts by explicit enumeration of distinct
  molecule instances over every (context, child) match, independent of the
  binomial formula and of the oracle's flattening loop.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import workloads as w


def test_paper_example_count_4_rate_4k():
    k = 0.375
    fm = oracle.FlatModel(w.paper_example_model(k=k))
    assert fm.M == 1
    e = fm.entries[0]
    assert e["context"] == 1 and e["child"] == -1
    a = oracle.propensities(fm, fm.desc["init"])
    assert a[0] == 4 * k
    # the first drawn step of the oracle uses the same rate
    r = oracle.simulate(fm.desc, 1, 1.0, 1.0, 1, trace_g=0, trace_cap=4, flat=fm)
    assert r["trace"][0][1] == 4 * k


@pytest.mark.parametrize("n,k,want", [(5, 2, 10), (2, 3, 0), (0, 0, 1), (7, 0, 1), (1000, 1, 1000)])
def test_binomial_spec_examples(n, k, want):
    assert oracle.binomial(n, k) == want


def test_binomial_matches_math_comb():
    rng = np.random.default_rng(0)
    for _ in range(500):
        n = int(rng.integers(0, 2**31))
        k = int(rng.integers(0, 3))
        assert oracle.binomial(n, k) == math.comb(n, k)
    assert oracle.binomial(64, 32) == math.comb(64, 32)


def test_match_populations_spec_examples():
    # {a:1,b:1} vs {a:2,b:2} -> 4 ; {} -> 1 ; {a:2} vs {a:5} -> 10
    def model(reactants, init):
        return w.models._flat_model("t", ["a", "b"], [w.models._rule(0, reactants, [], 1.0)], init)
    for re, init, want in [([(0, 0, 1), (0, 1, 1)], [2, 2], 4.0), ([], [3, 9], 1.0), ([(0, 0, 2)], [5, 0], 10.0)]:
        fm = oracle.FlatModel(model(re, init))
        assert oracle.propensities(fm, init)[0] == want


def test_label_mismatch_gives_no_entry():
    # rule labelled l applied to a term with only a TOP compartment -> empty matchset
    d = w.models._flat_model("t", ["a", "b"], [w.models._rule(1, [(0, 0, 1), (0, 1, 1)], [], 1.0)], [2, 2])
    d["n_types"] = 2
    assert oracle.FlatModel(d).M == 0


@pytest.mark.parametrize("sums,u,want", [([2, 3, 5], 0.45, 1), ([1, 0, 1], 0.6, 2), ([7.5], 0.999, 0),
                                         ([1, 0, 1], 0.49, 0), ([0, 0, 3], 0.0, 2)])
def test_selection_spec_examples(sums, u, want):
    a0 = float(sum(sums))
    assert oracle.select(sums, u * a0) == want


def test_selection_never_picks_zero_rate():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        a = rng.random(6) * (rng.random(6) < 0.5)
        if a.sum() == 0:
            continue
        a0 = 0.0
        for v in a:
            a0 = a0 + v
        mu = oracle.select(a, rng.random() * a0)
        assert a[mu] > 0


def _brute_counts(desc, x):
    """Per rule: total number of distinct reactant-instance combinations over
    all matches (context, child), by explicit enumeration of molecule ids."""
    S = desc["n_species"]
    parent, ctype = desc["parent"], desc["type"]
    C = len(parent)
    out = []
    for rule in desc["rules"]:
        total = 0
        for c in range(C):
            if ctype[c] != rule["label"]:
                continue
            kids = [None] if rule["child_label"] < 0 else [d for d in range(C) if parent[d] == c and ctype[d] == rule["child_label"]]
            for d in kids:
                # molecule instances: one id per molecule of each needed cell
                need = {}
                for (where, s, mult) in rule["reactants"]:
                    cell = (c if where == 0 else d) * S + s
                    need[cell] = need.get(cell, 0) + mult
                ways = 1
                for cell, mult in need.items():
                    ids = range(x[cell])
                    ways *= sum(1 for _ in itertools.combinations(ids, mult))
                total += ways
        out.append(total)
    return out


def test_flatten_counts_match_brute_force_enumeration():
    rng = np.random.default_rng(5)
    for trial in range(30):
        d = w.small_cwc_model(n_children=int(rng.integers(1, 4)), seed=trial)
        for r in d["rules"]:
            r["rate"] = 1.0
        x = [int(v) for v in rng.integers(0, 9, size=len(d["init"]))]
        fm = oracle.FlatModel(d)
        a = oracle.propensities(fm, x)
        per_rule = [0] * len(d["rules"])
        for e, v in zip(fm.entries, a):
            per_rule[e["rule"]] += int(v)
        assert per_rule == _brute_counts(d, x)


def test_flatten_order_and_sizes():
    fm = oracle.FlatModel(w.config("C5")[0])
    assert fm.M == 20 + 32 * 20 + 32 * 16 == 1172
    assert fm.n_cells == 33 * 8
    # rule-major, then context preorder, then child index
    keys = [(e["rule"], e["context"], e["child"]) for e in fm.entries]
    assert keys == sorted(keys)
    fm4 = oracle.FlatModel(w.config("C4")[0])
    assert fm4.M == 256 and fm4.n_cells == 64
    # transport entries move one molecule between parent and child
    tr = [e for e in fm.entries if e["child"] >= 0]
    assert len(tr) == 512
    for e in tr:
        assert sorted(d for _, d in e["nu"]) == [-1, 1]
