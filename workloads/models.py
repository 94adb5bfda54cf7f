"""Model descriptions and seeded generators for the five BASELINE.json configs
and the small models used by the oracle pins.

Sources: BASELINE.json `configs` (C1..C5) and SURVEY.md §8(c) readings 10-13
for the parts the configs leave open.  Nothing here computes any step of the
simulation method; it only states inputs.
"""
from __future__ import annotations

import json
import os

import numpy as np

_FROZEN = os.path.join(os.path.dirname(__file__), "frozen")


def _rule(label, reactants, products, rate, child_label=-1):
    return {
        "label": int(label),
        "child_label": int(child_label),
        "reactants": [tuple(int(v) for v in r) for r in reactants],
        "products": [tuple(int(v) for v in p) for p in products],
        "rate": float(rate),
    }


def _flat_model(name, species, rules, init, obs=None):
    """Single TOP compartment model; observables default to one per species."""
    S = len(species)
    if obs is None:
        obs = list(range(S))
    return {
        "name": name,
        "n_types": 1,
        "n_species": S,
        "species_names": list(species),
        "parent": [-1],
        "type": [0],
        "rules": rules,
        "init": [int(v) for v in init],
        "n_obs": max(obs) + 1 if obs else 0,
        "obs_of_cell": list(obs),
    }


# --------------------------------------------------------------------------
# Small models (oracle pins, parity cases)
# --------------------------------------------------------------------------

def decay_model(n0=1000, k=1.0):
    """A -> 0 at rate k*A."""
    return _flat_model("decay", ["A"], [_rule(0, [(0, 0, 1)], [], k)], [n0])


def immigration_death_model(k_in=10.0, k_out=0.1, a0=0):
    """0 -> A (k_in), A -> 0 (k_out*A) -- BASELINE.json configs[0]."""
    return _flat_model(
        "immigration_death",
        ["A"],
        [_rule(0, [], [(0, 0, 1)], k_in), _rule(0, [(0, 0, 1)], [], k_out)],
        [a0],
    )


def isomerisation_model(n=20, kf=1.0, kb=0.5, a0=None):
    """A -> B (kf*A), B -> A (kb*B); A + B = n is conserved."""
    a0 = n if a0 is None else a0
    return _flat_model(
        "isomerisation",
        ["A", "B"],
        [_rule(0, [(0, 0, 1)], [(0, 1, 1)], kf), _rule(0, [(0, 1, 1)], [(0, 0, 1)], kb)],
        [a0, n - a0],
    )


def dimerisation_model(a0=6, k=1.0):
    """A + A -> D, propensity k * C(A, 2) (P:637 binomial reading)."""
    return _flat_model(
        "dimerisation", ["A", "D"], [_rule(0, [(0, 0, 2)], [(0, 1, 1)], k)], [a0, 0]
    )


def lotka_volterra_model(k1=10.0, k2=0.01, k3=10.0, x0=1000, y0=1000):
    """X -> 2X (k1 X), X + Y -> 2Y (k2 X Y), Y -> 0 (k3 Y) -- configs[1]."""
    return _flat_model(
        "lotka_volterra",
        ["X", "Y"],
        [
            _rule(0, [(0, 0, 1)], [(0, 0, 2)], k1),
            _rule(0, [(0, 0, 1), (0, 1, 1)], [(0, 1, 2)], k2),
            _rule(0, [(0, 1, 1)], [], k3),
        ],
        [x0, y0],
    )


def lotka_volterra_chain(n, k1=10.0, k2=0.01, k3=10.0, x0=1000):
    """n-species Lotka-Volterra family (the workload of
    the paper's only numeric table, fig:simd:speedup P:687-706, whose
    parameters are not stated).  Reading: a predation chain
    X1 -> 2 X1 (k1 X1), Xi + Xi+1 -> 2 Xi+1 (k2 Xi Xi+1, i = 1..n-1),
    Xn -> 0 (k3 Xn); all Xi(0) = x0.  n = 2 is configs[1] (C2)."""
    rules = [_rule(0, [(0, 0, 1)], [(0, 0, 2)], k1)]
    for i in range(n - 1):
        rules.append(_rule(0, [(0, i, 1), (0, i + 1, 1)], [(0, i + 1, 2)], k2))
    rules.append(_rule(0, [(0, n - 1, 1)], [], k3))
    return _flat_model("lotka_volterra_%d" % n, ["X%d" % (i + 1) for i in range(n)], rules, [x0] * n)


def michaelis_menten_model(kf=1e-3, kr=1.0, kcat=0.1, e0=200, s0=1000):
    """E + S -> ES (kf), ES -> E + S (kr), ES -> E + P (kcat) -- configs[2]."""
    return _flat_model(
        "michaelis_menten",
        ["E", "S", "ES", "P"],
        [
            _rule(0, [(0, 0, 1), (0, 1, 1)], [(0, 2, 1)], kf),
            _rule(0, [(0, 2, 1)], [(0, 0, 1), (0, 1, 1)], kr),
            _rule(0, [(0, 2, 1)], [(0, 0, 1), (0, 3, 1)], kcat),
        ],
        [e0, s0, 0, 0],
    )


def mm_sweep(n_kf=64, n_kcat=64):
    """64x64 log-uniform grid: point p = n_kcat*a + b,
    kf_a = 10^(-4 + 3a/(n_kf-1)), kcat_b = 10^(-2 + 3b/(n_kcat-1)), endpoints
    inclusive.  Values are computed once here and passed to both sides."""
    values = []
    for a in range(n_kf):
        kf = 10.0 ** (-4.0 + 3.0 * a / (n_kf - 1)) if n_kf > 1 else 1e-4
        for b in range(n_kcat):
            kcat = 10.0 ** (-2.0 + 3.0 * b / (n_kcat - 1)) if n_kcat > 1 else 1e-2
            values.append([kf, kcat])
    return {"rules": [0, 2], "values": values}


def paper_example_model(k=0.5, label_child=True):
    """rule  l: a b X -> c X  applied to content  a a b b  of an
    l-type compartment; combination count 4, rate 4k.  The l-compartment is a
    child of TOP; the rule's label is l (type 1)."""
    S = 3  # a, b, c
    init = [0, 0, 0] + [2, 2, 0]
    rules = [_rule(1, [(0, 0, 1), (0, 1, 1)], [(0, 2, 1)], k)]
    return {
        "name": "paper_example",
        "n_types": 2,
        "n_species": S,
        "species_names": ["a", "b", "c"],
        "parent": [-1, 0],
        "type": [0, 1],
        "rules": rules,
        "init": init,
        "n_obs": 3,
        "obs_of_cell": [0, 1, 2, 0, 1, 2],
    }


def small_cwc_model(n_children=3, seed=7):
    """A small compartmented model (TOP + children, one grandchild) exercising
    every rule shape: local rules at both types, transport in/out through a
    child pattern, a child-pattern rule with reactants on both sides."""
    rng = np.random.default_rng(seed)
    S = 3
    parent = [-1] + [0] * n_children + [1]
    ctype = [0] + [1] * n_children + [1]
    C = len(parent)
    rules = [
        _rule(0, [], [(0, 0, 1)], 5.0),                       # TOP: 0 -> s0
        _rule(0, [(0, 0, 1)], [], 0.1),                       # TOP: s0 -> 0
        _rule(1, [(0, 1, 2)], [(0, 2, 1)], 0.01),             # C: s1 + s1 -> s2
        _rule(1, [(0, 2, 1)], [], 0.2),                       # C: s2 -> 0
        _rule(0, [(0, 0, 1)], [(1, 1, 1)], 0.05, child_label=1),   # s0@T -> s1@child
        _rule(0, [(1, 1, 1)], [(0, 0, 1)], 0.02, child_label=1),   # s1@child -> s0@T
        _rule(1, [(0, 2, 1), (1, 1, 1)], [(0, 1, 1), (1, 2, 1)], 0.003, child_label=1),
    ]
    init = [int(v) for v in rng.integers(0, 40, size=C * S)]
    obs = [ctype[c] * S + s for c in range(C) for s in range(S)]
    return {
        "name": "small_cwc",
        "n_types": 2,
        "n_species": S,
        "parent": parent,
        "type": ctype,
        "rules": rules,
        "init": init,
        "n_obs": 2 * S,
        "obs_of_cell": obs,
    }


# --------------------------------------------------------------------------
# Generators for C4 / C5 (frozen to JSON; the frozen file is the contract)
# --------------------------------------------------------------------------

def random_network_model(seed=1, n_species=64, n_reactions=256):
    """SURVEY §8(c).12 reading of configs[3]."""
    rng = np.random.default_rng(seed)
    rules = []
    for _ in range(n_reactions):
        order = int(rng.integers(0, 3))
        re = {}
        for _ in range(order):
            s = int(rng.integers(0, n_species))
            re[s] = re.get(s, 0) + 1
        n_prod = int(rng.integers(1, 3))
        pr = {}
        for _ in range(n_prod):
            s = int(rng.integers(0, n_species))
            st = int(rng.integers(1, 3))
            pr[s] = pr.get(s, 0) + st
        k = 10.0 ** rng.uniform(-4.0, 0.0)
        rules.append(_rule(0, [(0, s, m) for s, m in sorted(re.items())],
                           [(0, s, m) for s, m in sorted(pr.items())], k))
    init = [int(v) for v in rng.integers(100, 1001, size=n_species)]
    m = _flat_model("random_network", [f"s{i}" for i in range(n_species)], rules, init)
    m["generator"] = {"kind": "random_network", "seed": seed}
    return m


def cwc_compartment_model(seed=1, n_children=32, n_species=8):
    """SURVEY §8(c).13 reading of configs[4]."""
    rng = np.random.default_rng(seed)
    S = n_species
    half = S // 2
    rules = []
    for label in (0, 1):
        for i in range(S):
            rules.append(_rule(label, [], [(0, i, 1)], 10.0 ** rng.uniform(-3, 0)))
        for i in range(S):
            rules.append(_rule(label, [(0, i, 1)], [], 10.0 ** rng.uniform(-3, 0)))
        for i in range(half):
            rules.append(_rule(label, [(0, i, 2)], [(0, i + half, 1)], 10.0 ** rng.uniform(-3, 0)))
    for i in range(S):
        rules.append(_rule(0, [(0, i, 1)], [(1, i, 1)], 10.0 ** rng.uniform(-3, 0), child_label=1))
    for i in range(S):
        rules.append(_rule(0, [(1, i, 1)], [(0, i, 1)], 10.0 ** rng.uniform(-3, 0), child_label=1))
    parent = [-1] + [0] * n_children
    ctype = [0] + [1] * n_children
    C = len(parent)
    init = [int(v) for v in rng.integers(0, 501, size=C * S)]
    obs = [ctype[c] * S + s for c in range(C) for s in range(S)]
    return {
        "name": "cwc_compartments",
        "n_types": 2,
        "n_species": S,
        "species_names": [f"s{i}" for i in range(S)],
        "parent": parent,
        "type": ctype,
        "rules": rules,
        "init": init,
        "n_obs": 2 * S,
        "obs_of_cell": obs,
        "generator": {"kind": "cwc_compartments", "seed": seed},
    }


def _load_frozen(name, gen):
    path = os.path.join(_FROZEN, name + ".json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        for r in m["rules"]:
            r["reactants"] = [tuple(v) for v in r["reactants"]]
            r["products"] = [tuple(v) for v in r["products"]]
        return m
    return gen()


def freeze_all():
    """Write the C4/C5 generator output to workloads/frozen/ (run once)."""
    os.makedirs(_FROZEN, exist_ok=True)
    for name, gen in (("c4_random_network", random_network_model),
                      ("c5_cwc_compartments", cwc_compartment_model)):
        with open(os.path.join(_FROZEN, name + ".json"), "w") as f:
            json.dump(gen(), f, indent=1)


# --------------------------------------------------------------------------
# The five configs (BASELINE.json "configs")
# --------------------------------------------------------------------------

CONFIGS = {
    "C1": dict(desc="immigration-death", t_end=100.0, sample_dt=1.0, n_replicas=1024, seed=1),
    "C2": dict(desc="lotka-volterra", t_end=10.0, sample_dt=0.01, n_replicas=16384, seed=1),
    "C3": dict(desc="michaelis-menten 64x64 sweep", t_end=50.0, sample_dt=0.5, n_replicas=16, seed=1),
    "C4": dict(desc="random 64 species / 256 reactions", t_end=1.0, sample_dt=0.01, n_replicas=32768, seed=1),
    "C5": dict(desc="CWC 1+32 compartments", t_end=20.0, sample_dt=0.1, n_replicas=8192, seed=1),
}


def config(name):
    """Return (model_desc, sweep_or_None, run_params) for config C1..C5."""
    p = dict(CONFIGS[name])
    if name == "C1":
        return immigration_death_model(), None, p
    if name == "C2":
        return lotka_volterra_model(), None, p
    if name == "C3":
        return michaelis_menten_model(), mm_sweep(), p
    if name == "C4":
        return _load_frozen("c4_random_network", random_network_model), None, p
    if name == "C5":
        return _load_frozen("c5_cwc_compartments", cwc_compartment_model), None, p
    raise KeyError(name)
