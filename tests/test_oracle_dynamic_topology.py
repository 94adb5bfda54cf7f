"""Pins of the dynamic-topology CWC oracle (oracle/dynamic.py, SURVEY 8(f)
NEXT-4): compartments created, deleted, dissolved and rewritten by rules.

  * reduction: every fixed-tree model (its rules rewrite children in place)
    gives exactly the trajectories of the fixed-tree oracle oracle.simulate
    (itself pinned by closed forms, CME and the Philox library KATs);
  * Match_Populations x count_compartments equals a
    brute-force count of distinct reactant choices over individually named
    molecules, contexts and children, on random small terms;
  * closed forms of dynamic topologies: compartment immigration-death
    (creation at rate lam, deletion at rate mu per compartment: the number of
    compartments is Poisson(lam/mu (1 - e^{-mu t}))); dissolution releasing a
    molecule carried inside (top-level count Poisson(lam t - lam/delta
    (1 - e^{-delta t})), whole-term count Poisson(lam t));
  * stoichiometry of every firing along a trace (whole-term totals change by
    exactly the rule's net change, compartments by its creations/deletions).
"""
import itertools
import math
import random

import numpy as np
import pytest

import oracle
import workloads as w
from oracle import dynamic as dyn


def _preorder_cwc(seed=3):
    """A small CWC tree in preorder index order (a grandchild right after its
    parent), with every fixed-tree rule shape: local, transport both ways,
    child-pattern rule with reactants on both sides, A + A."""
    d = w.small_cwc_model(3, seed)
    d["parent"] = [-1, 0, 1, 0, 0]
    return d


FIXED = [("paper", lambda: w.paper_example_model(0.5), dict(t_end=5.0, sample_dt=0.5, n_replicas=24, seed=2)),
         ("C1", lambda: w.config("C1")[0], dict(t_end=20.0, sample_dt=1.0, n_replicas=16, seed=1)),
         ("C2", lambda: w.config("C2")[0], dict(t_end=0.03, sample_dt=0.01, n_replicas=6, seed=1)),
         ("dimer", lambda: w.dimerisation_model(30, 0.2), dict(t_end=2.0, sample_dt=0.1, n_replicas=16, seed=8)),
         ("stall", lambda: w.decay_model(3, 5.0), dict(t_end=10.0, sample_dt=1.0, n_replicas=16, seed=4)),
         ("cwc", _preorder_cwc, dict(t_end=0.5, sample_dt=0.05, n_replicas=10, seed=5))]


@pytest.mark.parametrize("name,make,cfg", FIXED, ids=[f[0] for f in FIXED])
def test_fixed_tree_models_reduce_to_the_fixed_oracle(name, make, cfg):
    desc = make()
    m = dyn.from_fixed_tree(desc)
    a = dyn.simulate(m, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
    b = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], want_stats=False)
    assert np.array_equal(a["traj"], b["traj"])
    assert np.array_equal(a["firings"], b["firings"])
    assert np.array_equal(a["status"], b["status"])


def test_paper_example_rate():
    # rule l: a b X -> c X on content a a b b of an l-compartment: 4 combinations
    term = dyn.term_from_spec({"comps": [{"label": 1, "content": {"atoms": {"a": 2, "b": 2}}}]})
    rule = {"label": 1, "atoms": {"a": 1, "b": 1}, "rate": 0.5, "rhs": {"X": True, "atoms": {"c": 1}}}
    e = dyn.match_entries([rule], term)
    assert len(e) == 1 and e[0][3] == 4 and rule["rate"] * e[0][3] == 2.0
    # the same rule at the top level (label mismatch): no entry
    top = dyn.term_from_spec({"atoms": {"a": 2, "b": 2}})
    assert dyn.match_entries([rule], top) == []


def _tokens(ms, tag):
    return [(tag, a, i) for a, n in ms.items() for i in range(n)]


def _brute(rule, term):
    """Distinct reactant choices over individually named molecules."""
    out = []
    for lab, t in dyn._contexts(term):
        if lab != rule["label"]:
            continue
        ctx_tok = _tokens(t.atoms, "c")

        def choices(tokens, pattern):
            k = sum(pattern.values())
            cnt = 0
            for sub in itertools.combinations(tokens, k):
                got = {}
                for (_, a, _) in sub:
                    got[a] = got.get(a, 0) + 1
                cnt += got == {a: m for a, m in pattern.items() if m}
            return cnt
        hc = choices(ctx_tok, rule.get("atoms", {}))
        cp = rule.get("comp")
        if cp is None:
            out.append(hc)
            continue
        for c in t.comps:
            if c.label == cp["label"]:
                out.append(hc * choices(_tokens(c.wrap, "w"), cp.get("wrap", {})) *
                           choices(_tokens(c.content.atoms, "y"), cp.get("content", {})))
    return out


def _random_term(rng, depth=2):
    atoms = {a: rng.randrange(0, 4) for a in "abc" if rng.random() < 0.8}
    comps = []
    if depth > 0:
        for _ in range(rng.randrange(0, 3)):
            comps.append({"label": rng.randrange(1, 3), "wrap": {a: rng.randrange(0, 3) for a in "rs"},
                          "content": _random_term(rng, depth - 1)})
    return {"atoms": atoms, "comps": comps}


def test_match_counts_equal_brute_force_enumeration():
    rng = random.Random(11)
    rules = [{"label": 0, "atoms": {"a": 1, "b": 1}, "rate": 1.0, "rhs": {}},
             {"label": 1, "atoms": {"a": 2}, "rate": 1.0, "rhs": {}},
             {"label": 0, "atoms": {"c": 1}, "comp": {"label": 1, "wrap": {"r": 1}, "content": {"a": 1}}, "rate": 1.0,
              "rhs": {}},
             {"label": 1, "atoms": {}, "comp": {"label": 2, "wrap": {"r": 1, "s": 2}, "content": {"b": 2}}, "rate": 1.0,
              "rhs": {}},
             {"label": 2, "atoms": {"a": 1, "c": 2}, "comp": {"label": 1, "wrap": {}, "content": {}}, "rate": 1.0,
              "rhs": {}}]
    for _ in range(60):
        term = dyn.term_from_spec(_random_term(rng))
        for ri, r in enumerate(rules):
            got = [e[3] for e in dyn.match_entries([r], term)]
            assert got == _brute(r, term), (ri,)


# ---- dynamic topologies: closed forms --------------------------------------

def _z_ok(samples, mean, var, z=4.5):
    """|sample mean - mean| within z standard errors (Bonferroni-safe z)."""
    n = len(samples)
    return abs(samples.mean() - mean) <= z * math.sqrt(var / n) + 1e-12


def test_compartment_immigration_death_is_poisson():
    lam, mu = 6.0, 0.5
    model = {"term": {},
             "rules": [{"label": 0, "atoms": {}, "rate": lam, "rhs": {"X": True, "comps": [{"label": 1}]}},
                       {"label": 0, "atoms": {}, "comp": {"label": 1, "wrap": {}, "content": {}}, "rate": mu,
                        "rhs": {"X": True}}],
             "observables": [("count", 1)]}
    T, dt = 4.0, 1.0
    r = dyn.simulate(model, 1500, T, dt, 7)
    for j in range(1, 5):
        m = lam / mu * (1 - math.exp(-mu * j * dt))
        x = r["traj"][:, j, 0].astype(float)
        assert _z_ok(x, m, m), (j, x.mean(), m)
        # Poisson: variance = mean (chi-square-free check: within 20 %)
        assert abs(x.var(ddof=1) / m - 1.0) < 0.2, (j, x.var(), m)


def test_dissolution_releases_content():
    lam, delta = 5.0, 0.8
    model = {"term": {},
             "rules": [{"label": 0, "atoms": {}, "rate": lam,
                        "rhs": {"X": True, "comps": [{"label": 1, "content": {"a": 1}}]}},
                       {"label": 0, "atoms": {}, "comp": {"label": 1, "wrap": {}, "content": {}}, "rate": delta,
                        "rhs": {"X": True, "release_Y": True}}],
             "observables": [("content", 0, "a"), [("content", 0, "a"), ("content", 1, "a")], ("count", 1)]}
    T, dt = 3.0, 1.0
    r = dyn.simulate(model, 1500, T, dt, 9)
    for j in range(1, 4):
        t = j * dt
        m_top = lam * t - lam / delta * (1 - math.exp(-delta * t))
        assert _z_ok(r["traj"][:, j, 0].astype(float), m_top, m_top), j
        assert _z_ok(r["traj"][:, j, 1].astype(float), lam * t, lam * t), j
        # every live compartment carries exactly one a
        assert (r["traj"][:, j, 1] - r["traj"][:, j, 0] == r["traj"][:, j, 2]).all()


def test_stoichiometry_along_a_trace():
    """A model with creation, in-place rewriting with wrap changes, transport,
    dissolution and deletion: whole-term totals change by exactly each fired
    rule's net change."""
    rules = [
        {"label": 0, "atoms": {"a": 1}, "rate": 2.0, "rhs": {"X": True, "comps": [{"label": 1, "wrap": {"r": 1},
                                                                                   "content": {"b": 2}}]}},
        {"label": 0, "atoms": {"a": 1}, "comp": {"label": 1, "wrap": {"r": 1}, "content": {}}, "rate": 0.3,
         "rhs": {"X": True, "comps": [{"label": 1, "W": True, "Y": True, "wrap": {"r": 1}, "content": {"a": 1}}]}},
        {"label": 1, "atoms": {"b": 1}, "rate": 0.5, "rhs": {"X": True, "atoms": {"c": 1}}},
        {"label": 0, "atoms": {}, "comp": {"label": 1, "wrap": {"r": 2}, "content": {"c": 1}}, "rate": 0.2,
         "rhs": {"X": True, "release_Y": True, "atoms": {"a": 1}}},
        {"label": 0, "atoms": {}, "comp": {"label": 1, "wrap": {}, "content": {}}, "rate": 0.05, "rhs": {"X": True}},
        {"label": 0, "atoms": {}, "rate": 1.0, "rhs": {"X": True, "atoms": {"a": 1}}},
    ]
    # net change of (a, b, c, r, count) for the rules whose effect does not depend on the match
    net = {0: (-1, 2, 0, 1, 1), 1: (0, 0, 0, 0, 0), 2: (0, -1, 1, 0, 0), 5: (1, 0, 0, 0, 0)}
    model = {"term": {"atoms": {"a": 5}}, "rules": rules,
             "observables": [[("content", 0, "a"), ("content", 1, "a")], [("content", 0, "b"), ("content", 1, "b")],
                             [("content", 0, "c"), ("content", 1, "c")], ("wrap", 1, "r"), ("count", 1)]}
    for g in range(4):
        trace = []
        term = dyn.term_from_spec(model["term"])
        prev = dyn.observe(term, model["observables"])
        _, fir, st = dyn.simulate_one(model, g, 5.0, 5.0, 3, trace=trace)
        # replay the trace on a fresh term and check every step's change
        term = dyn.term_from_spec(model["term"])
        for rec in trace:
            mu = int(rec[4])
            if mu < 0:
                break
            entries = dyn.match_entries(rules, term)
            ri, ctx, ci, h = entries[mu]
            assert h > 0
            dyn.apply_rule(rules[ri], ctx, ci)
            cur = dyn.observe(term, model["observables"])
            d = tuple(c - p for c, p in zip(cur, prev))
            if ri in net:
                assert d == net[ri], (ri, d)
            elif ri == 3:  # dissolution: c moves to the top, r (2) dropped with the wrap, +a, -1 compartment
                assert d[2] == 0 and d[3] <= -2 and d[4] == -1 and d[0] >= 1
            elif ri == 4:  # deletion: the compartment and everything in it vanish
                assert d[4] == -1 and d[0] <= 0 and d[1] <= 0 and d[2] <= 0 and d[3] <= 0
            prev = cur
        assert len([r for r in trace if r[4] >= 0]) == fir


@pytest.mark.parametrize("top,expect_status", [(2**31 - 2, 1), (2**31 - 1, 2)])
def test_release_overflow_freezes_before_the_update(top, expect_status):
    """Reading 7 (OVERFLOW) on a dissolution: releasing the child's single a
    into a top level holding `top` of them either fits in int32 (the rule
    fires once, then the term stalls with 2^31-1) or would not (the term
    freezes before the update: status OVERFLOW, every sample the initial
    state)."""
    model = {"term": {"atoms": {"a": top}, "comps": [{"label": 1, "content": {"atoms": {"a": 1}}}]},
             "rules": [{"label": 0, "atoms": {}, "comp": {"label": 1, "wrap": {}, "content": {}}, "rate": 1.0,
                        "rhs": {"X": True, "release_Y": True}}],
             "observables": [("content", 0, "a"), ("count", 1)]}
    samples, fir, st = dyn.simulate_one(model, 0, 50.0, 10.0, 1)
    assert st == expect_status
    if expect_status == 1:
        assert fir == 1 and samples[-1].tolist() == [2**31 - 1, 0]
    else:
        assert fir == 0 and (samples == [top, 1]).all()
