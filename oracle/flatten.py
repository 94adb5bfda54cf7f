"""Oracle flattening of CWC rules over a FIXED compartment tree.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

Follows PAPER.md Fig. `fig:simd`: `Simulation_Step` iterates
"foreach r in ruleset" and `Match(rule, term, context)` visits the
top level and then recurses into every compartment content; a
rule with label l applies only in contexts of type l.  With a
fixed tree the recursion visits compartments in preorder; this oracle requires
parent[c] < c and uses compartment index order as that preorder
(SURVEY §8(c) "flatten").  One flat reaction ("entry") is emitted per
(rule, context) -- and, for a rule whose pattern contains a child compartment
of type child_label, per (rule, context, child) with children in index order
(the `count_compartments` factor of P:627 expanded into one entry per matched
child).

Each entry carries:
  reactants: list of (cell, mult) with cell = compartment * n_species + species,
             duplicates merged (a pattern is a multiset);
  nu:        {cell: products - reactants}, zero entries dropped;
  rule:      the rule index, which selects the rate constant k.
"""
from __future__ import annotations


def flatten(desc):
    S = int(desc["n_species"])
    parent = [int(v) for v in desc["parent"]]
    ctype = [int(v) for v in desc["type"]]
    C = len(parent)
    assert parent[0] == -1 and ctype[0] == 0
    for c in range(1, C):
        assert 0 <= parent[c] < c, "oracle requires parent[c] < c (preorder numbering)"
    children = [[d for d in range(C) if parent[d] == c] for c in range(C)]

    entries = []
    for r, rule in enumerate(desc["rules"]):                 # foreach r in ruleset
        for c in range(C):                                    # Match recursion, preorder
            if ctype[c] != rule["label"]:
                continue
            if rule["child_label"] < 0:
                contexts = [(c, None)]
            else:
                contexts = [(c, d) for d in children[c] if ctype[d] == rule["child_label"]]
            for (ctx, child) in contexts:
                def cell(where, s):
                    comp = ctx if where == 0 else child
                    assert comp is not None, "child reactant on a local rule"
                    return comp * S + s

                re = {}
                for (where, s, mult) in rule["reactants"]:
                    k = cell(where, s)
                    re[k] = re.get(k, 0) + mult
                pr = {}
                for (where, s, mult) in rule["products"]:
                    k = cell(where, s)
                    pr[k] = pr.get(k, 0) + mult
                nu = {}
                for k in sorted(set(re) | set(pr)):
                    d = pr.get(k, 0) - re.get(k, 0)
                    if d != 0:
                        nu[k] = d
                entries.append({
                    "rule": r,
                    "context": ctx,
                    "child": -1 if child is None else child,
                    "reactants": sorted(re.items()),
                    "nu": sorted(nu.items()),
                })
    return entries
