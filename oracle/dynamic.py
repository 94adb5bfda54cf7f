"""CPU oracle of dynamic-topology CWC: terms whose
compartments are created, dissolved, deleted and rewritten by the rules.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain, slow, pure
Python: for the small cases of its pins.  Random numbers, uniforms and tau
come from the oracle's C functions (oracle.philox4x32_10, oracle.uniforms,
oracle.tau) so that a fixed-topology model gives exactly the trajectories of
oracle.simulate (the reduction pin in tests/test_oracle_dynamic.py).

The calculus:
  * a term is a multiset of atoms and compartments (wrap | content)^label
    (P:158-167): here a Term holds an atom multiset and an ordered list of
    Comp(label, wrap multiset, content Term); the top level is a Term with
    label 0 (TOP);
  * a rule  label: P --k--> O with P = context atoms +
    the rest variable X + at most ONE compartment pattern
    (label', wrap atoms + wrap rest W | content atoms + content rest Y),
    depth 1 (SPEC S:38-49, S:146 design decisions);
  * O = atoms, optionally X (the context's rest is kept; without X it is
    deleted: sigma(O) replaces the whole matched content u),
    optionally Y / W released into the context (dissolution), and compartment
    constructors (label'', atoms + optionally W | atoms + optionally Y).

Readings where the paper is silent:
  D1 matching and rates: for each rule, each context (the top level for
     TOP rules, every compartment of the rule's label, in PREORDER of the
     current term), and -- with a compartment pattern -- each child of the
     context with label' in list order, one match entry with rate
     k * RN(h), h = prod binomial(n, mult) over the context atoms, the
     child's wrap atoms and the child's content atoms, exact integers
     (Fig. fig:simd P:623-640: count_population *
     count_compartments * k);
  D2 one flat selection over the entries in that order (reading 2 of the
     fixed-tree oracle), one Philox block per loop iteration keyed (n, g);
  D3 update: remove P's atoms from the context; a matched child is removed
     from the context's list, binding W = wrap - pattern wrap atoms and Y =
     content - pattern content atoms (its sub-compartments stay in Y);
     without X the rest of the context (atoms and compartments) is deleted;
     O's atoms are added, released W / Y merge into the context (Y's
     compartments appended), constructors create compartments: one that
     carries BOTH W and Y of the matched child takes that child's position in
     the list (the compartment is rewritten in place, keeping its identity),
     any other constructor is appended;  W and Y are each used at most once;
  D4 observables: ("content", label, atom) = total count of atom in the
     contents of all compartments of that label (label 0: the top level),
     ("wrap", label, atom), ("count", label) = number of compartments of
     that label; samples take the pre-event state at t_j = j dt (the fixed
     oracle's sampling, termination and stall rules).
"""
from __future__ import annotations

import math

import numpy as np

from . import philox4x32_10, tau as oracle_tau, uniforms

INT32_MAX = 2**31 - 1


class Term:
    __slots__ = ("atoms", "comps")

    def __init__(self, atoms=None, comps=None):
        self.atoms = {a: n for a, n in (atoms or {}).items() if n}
        self.comps = list(comps or [])

    def copy(self):
        return Term(dict(self.atoms), [c.copy() for c in self.comps])


class Comp:
    __slots__ = ("label", "wrap", "content")

    def __init__(self, label, wrap=None, content=None):
        self.label = int(label)
        self.wrap = {a: n for a, n in (wrap or {}).items() if n}
        self.content = content if content is not None else Term()

    def copy(self):
        return Comp(self.label, dict(self.wrap), self.content.copy())


def term_from_spec(spec):
    """spec: {"atoms": {a: n}, "comps": [{"label": l, "wrap": {...}, "content": spec}, ...]}"""
    return Term(dict(spec.get("atoms", {})),
                [Comp(c["label"], dict(c.get("wrap", {})), term_from_spec(c.get("content", {})))
                 for c in spec.get("comps", [])])


def _binomial(n, k):
    return math.comb(n, k) if 0 <= k <= n else 0


def _pop(pattern, multiset):
    """Match_Populations (Fig. fig:simd P:633-640): prod binomial(n_x, k_x)."""
    h = 1
    for a, k in pattern.items():
        h *= _binomial(multiset.get(a, 0), k)
        if h == 0:
            return 0
    return h


def _contexts(term):
    """(label, Term) of the top level and every compartment's content, in preorder."""
    out = [(0, term)]

    def rec(t):
        for c in t.comps:
            out.append((c.label, c.content))
            rec(c.content)
    rec(term)
    return out


def match_entries(rules, term):
    """D1: [(rule index, context Term, child index or -1, h)] in canonical order."""
    ctx = _contexts(term)
    entries = []
    for ri, r in enumerate(rules):
        for lab, t in ctx:
            if lab != r["label"]:
                continue
            hp = _pop(r.get("atoms", {}), t.atoms)
            cp = r.get("comp")
            if cp is None:
                entries.append((ri, t, -1, hp))
                continue
            for ci, c in enumerate(t.comps):
                if c.label != cp["label"]:
                    continue
                h = hp * _pop(cp.get("wrap", {}), c.wrap) * _pop(cp.get("content", {}), c.content.atoms)
                entries.append((ri, t, ci, h))
    return entries


def _sub(ms, pattern):
    for a, k in pattern.items():
        v = ms.get(a, 0) - k
        assert v >= 0, "pattern does not match"
        if v:
            ms[a] = v
        else:
            ms.pop(a, None)


def _add(ms, extra):
    for a, k in extra.items():
        if k:
            ms[a] = ms.get(a, 0) + k


def apply_rule(rule, t, ci):
    """D3: rewrite context Term t in place with rule, matched child index ci (or -1)."""
    _sub(t.atoms, rule.get("atoms", {}))
    W = Y = None
    pos = None
    if ci >= 0:
        c = t.comps.pop(ci)
        pos = ci
        W = dict(c.wrap)
        _sub(W, rule["comp"].get("wrap", {}))
        Y = c.content
        _sub(Y.atoms, rule["comp"].get("content", {}))
    rhs = rule["rhs"]
    if not rhs.get("X", True):
        t.atoms = {}
        t.comps = []
        pos = 0
    _add(t.atoms, rhs.get("atoms", {}))
    used_w = used_y = 0
    if rhs.get("release_W") and W is not None:
        _add(t.atoms, W)
        used_w += 1
    if rhs.get("release_Y") and Y is not None:
        _add(t.atoms, Y.atoms)
        t.comps.extend(Y.comps)
        used_y += 1
    for k in rhs.get("comps", []):
        wrap = dict(k.get("wrap", {}))
        content = Term(dict(k.get("content", {})))
        if k.get("W") and W is not None:
            _add(wrap, W)
            used_w += 1
        if k.get("Y") and Y is not None:
            _add(content.atoms, Y.atoms)
            content.comps = list(Y.comps)
            used_y += 1
        nc = Comp(k["label"], wrap, content)
        if k.get("W") and k.get("Y") and pos is not None:
            t.comps.insert(pos, nc)  # rewritten in place (keeps its list position)
            pos = None
        else:
            t.comps.append(nc)
    assert used_w <= 1 and used_y <= 1, "W and Y are each used at most once (reading D3)"


def _observe_one(term, ob):
    kind = ob[0]
    v = 0
    if kind == "content":
        _, lab, a = ob
        for l2, t in _contexts(term):
            if l2 == lab:
                v += t.atoms.get(a, 0)
    elif kind == "wrap":
        _, lab, a = ob
        stack = [term]
        while stack:
            t = stack.pop()
            for c in t.comps:
                if c.label == lab:
                    v += c.wrap.get(a, 0)
                stack.append(c.content)
    elif kind == "count":
        lab = ob[1]
        stack = [term]
        while stack:
            t = stack.pop()
            for c in t.comps:
                v += c.label == lab
                stack.append(c.content)
    else:
        raise ValueError(ob)
    return v


def observe(term, observables):
    """D4: observable values of the whole term; an observable is one key or a
    list of keys whose values are summed."""
    vals = []
    for ob in observables:
        keys = ob if isinstance(ob, list) else [ob]
        vals.append(sum(_observe_one(term, k) for k in keys))
    return vals


def _max_count(term):
    m = max(term.atoms.values(), default=0)
    for c in term.comps:
        m = max(m, max(c.wrap.values(), default=0), _max_count(c.content))
    return m


def simulate_one(model, g, t_end, dt, seed, trace=None):
    """One trajectory g (loop of P:608-621 / the fixed oracle's, D1-D4).
    model: {"term": spec, "rules": [...], "observables": [...], "rates": optional override list}.
    Returns (samples [J+1][O] int64, firings, status)."""
    rules = model["rules"]
    obs = model["observables"]
    term = term_from_spec(model["term"])
    J = int(math.floor(t_end / dt))
    samples = np.zeros((J + 1, len(obs)), dtype=np.int64)
    t, n, j, firings = 0.0, 0, 0, 0
    key = [seed & 0xFFFFFFFF, seed >> 32]
    while True:
        entries = match_entries(rules, term)
        rates = [rules[e[0]]["rate"] * float(e[3]) for e in entries]
        a0 = 0.0
        for i, r in enumerate(rates):
            a0 = r if i == 0 else a0 + r
        if a0 == 0.0:  # stall
            v = observe(term, obs)
            while j <= J:
                samples[j] = v
                j += 1
            return samples, firings, 1
        w = philox4x32_10([n & 0xFFFFFFFF, n >> 32, g & 0xFFFFFFFF, g >> 32], key)
        n += 1
        u1, u2 = uniforms(w)
        tau = oracle_tau(u1, a0)
        tn = t + tau
        if j <= J and j * dt <= tn:
            v = observe(term, obs)
            while j <= J and j * dt <= tn:
                samples[j] = v
                j += 1
        if j > J:
            if trace is not None:
                trace.append((n - 1, a0, tau, tn, -1))
            return samples, firings, 0
        target = u2 * a0
        c = 0.0
        mu = -1
        for i, r in enumerate(rates):
            c = c + r
            if target < c:
                mu = i
                break
        if mu < 0:
            mu = max(i for i, r in enumerate(rates) if r > 0.0)
        if trace is not None:
            trace.append((n - 1, a0, tau, tn, mu))
        ri, ctx, ci, _ = entries[mu]
        trial = term.copy() if _might_overflow(rules[ri]) else None
        apply_rule(rules[ri], ctx, ci)
        if trial is not None and _max_count(term) > INT32_MAX:  # freeze before the update
            term = trial
            v = observe(term, obs)
            while j <= J:
                samples[j] = v
                j += 1
            return samples, firings, 2
        t = tn
        firings += 1


def _might_overflow(rule):
    """Whether a firing can raise a count (so the OVERFLOW rule, reading 7,
    must look at the result): O's atoms, constructor atoms, or W / Y
    released into the context (dissolution adds the child's counts to the
    context's)."""
    rhs = rule["rhs"]
    released = rule.get("comp") is not None and (rhs.get("release_W") or rhs.get("release_Y"))
    return (bool(rhs.get("atoms")) or bool(released)
            or any(k.get("wrap") or k.get("content") for k in rhs.get("comps", [])))


def simulate(model, n_replicas, t_end, dt, seed, g_list=None):
    """Trajectories g_list (default all) -> dict(traj [n][J+1][O], firings, status)."""
    g_list = list(range(n_replicas)) if g_list is None else list(g_list)
    out = [simulate_one(model, g, t_end, dt, seed) for g in g_list]
    return dict(traj=np.stack([o[0] for o in out]), firings=np.array([o[1] for o in out]),
                status=np.array([o[2] for o in out]))


def from_fixed_tree(desc):
    """A fixed-tree model description (workloads format) as a dynamic model:
    compartment index order must be the preorder (parent[c] < c and every
    subtree contiguous).  Child-pattern rules rewrite the child in place
    (W and Y kept), so the topology never changes."""
    S = int(desc["n_species"])
    parent, ctype = desc["parent"], desc["type"]
    C = len(parent)
    kids = [[] for _ in range(C)]
    for c in range(1, C):
        kids[parent[c]].append(c)
    # preorder check
    order = []

    def rec(c):
        order.append(c)
        for k in kids[c]:
            rec(k)
    rec(0)
    assert order == list(range(C)), "compartment index order is not the preorder"

    def spec(c):
        return {"atoms": {s: desc["init"][c * S + s] for s in range(S)},
                "comps": [{"label": ctype[k], "wrap": {}, "content": spec(k)} for k in kids[c]]}

    rules = []
    for r in desc["rules"]:
        ctx_re = {}
        ch_re = {}
        for (wh, s, m) in r["reactants"]:
            d = ch_re if wh else ctx_re
            d[s] = d.get(s, 0) + m
        ctx_pr = {}
        ch_pr = {}
        for (wh, s, m) in r["products"]:
            d = ch_pr if wh else ctx_pr
            d[s] = d.get(s, 0) + m
        rule = {"label": r["label"], "atoms": ctx_re, "rate": float(r["rate"]),
                "rhs": {"X": True, "atoms": ctx_pr}}
        if r["child_label"] >= 0:
            rule["comp"] = {"label": r["child_label"], "wrap": {}, "content": ch_re}
            rule["rhs"]["comps"] = [{"label": r["child_label"], "W": True, "Y": True, "content": ch_pr}]
        rules.append(rule)
    n_obs = int(desc["n_obs"])
    # observable o = sum of its cells, as a sum of per-(type, species) totals:
    # every cell of a (type, species) pair must belong to the same observable
    keys = [set() for _ in range(n_obs)]
    owner = {}
    for cell, o in enumerate(desc["obs_of_cell"]):
        key = ("content", ctype[cell // S], cell % S)
        assert owner.setdefault(key, o) == o, "observables must be unions of per-type species totals"
        if o >= 0:
            keys[o].add(key)
    obs = [sorted(k) for k in keys]
    return {"term": spec(0), "rules": rules, "observables": obs}
