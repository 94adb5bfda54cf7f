"""Dynamic-topology CWC model descriptions.

Inputs only (no arithmetic of the method).  Format = oracle/dynamic.py's
model dict, which the CUDA side's binding (cwc.dyn_model_create) also reads:

    term  = {"atoms": {atom: n}, "comps": [{"label", "wrap": {atom: n},
             "content": term}, ...]}             the initial term
    rules = [{"label": context label,
              "atoms": {atom: mult},             context atoms of the pattern P
              "comp": {"label", "wrap": {..}, "content": {..}}   optional child pattern
              "rate": k,
              "rhs": {"X": keep the context's rest (default True),
                      "atoms": {..},             atoms of O added to the context
                      "release_W", "release_Y": the matched child's rest
                                                 variables released into the context,
                      "comps": [{"label", "wrap", "content", "W", "Y"}]}}]
                                                 compartment constructors of O
    observables = [key or [keys]]  key = ("content" | "wrap", label, atom)
                                   or ("count", label)

Atoms are small integers (0 .. n_atoms-1); label 0 is TOP.
"""
from __future__ import annotations

import random

# atoms of the cell-population model
N, A, R, B, P = 0, 1, 2, 3, 4
TOP, CELL, VES = 0, 1, 2
ATOM_NAMES = ["n", "a", "r", "b", "p"]
LABEL_NAMES = ["TOP", "CELL", "VES"]


def _r(label, rate, atoms=None, comp=None, X=True, rhs_atoms=None, release_W=False, release_Y=False, comps=None):
    rule = {"label": label, "atoms": dict(atoms or {}), "rate": float(rate),
            "rhs": {"X": X, "atoms": dict(rhs_atoms or {}), "release_W": release_W, "release_Y": release_Y,
                    "comps": list(comps or [])}}
    if comp is not None:
        rule["comp"] = comp
    return rule


def _pat(label, wrap=None, content=None):
    return {"label": label, "wrap": dict(wrap or {}), "content": dict(content or {})}


def _ctor(label, wrap=None, content=None, W=False, Y=False):
    return {"label": label, "wrap": dict(wrap or {}), "content": dict(content or {}), "W": W, "Y": Y}


def cell_population_model(n_cells=16, n0=400, a0=6, r0=3, scale=1.0):
    """C6: a population of cells (label CELL) in a nutrient bath (TOP) that
    take up nutrient through membrane receptors, divide, die by lysis
    (releasing membrane and content -- with any vesicles inside -- into the
    bath), and form vesicles (label VES, nested inside cells: depth 2) that
    later fuse back.  Every rule shape of the dynamic calculus occurs:
    local rules at three context labels, in-place rewriting of a child
    (uptake, receptor expression and turnover, export), creation by an
    appended constructor (division, vesicle formation), dissolution
    releasing W and Y (lysis; sub-compartments move up one level), release of
    Y only (fusion), deletion of a matched child (vesicle decay), and
    rules without X (a vesicle collapsing, a cell's clear-out: the rest of
    the context -- atoms and compartments -- is deleted).  Rates are the
    stochastic constants directly (reading 1)."""
    s = float(scale)
    rules = [
        _r(TOP, 60.0 * s, rhs_atoms={N: 1}),                                     # 0 nutrient influx
        _r(TOP, 0.05 * s, atoms={N: 1}),                                         # 1 nutrient decay
        _r(TOP, 0.002 * s, atoms={N: 1}, comp=_pat(CELL, wrap={R: 1}),           # 2 uptake through a receptor
           comps=[_ctor(CELL, wrap={R: 1}, content={N: 1}, W=True, Y=True)]),
        _r(CELL, 0.5 * s, atoms={N: 1}, rhs_atoms={A: 1}),                       # 3 metabolism
        _r(TOP, 0.02 * s, comp=_pat(CELL, content={A: 1}),                       # 4 receptor expression
           comps=[_ctor(CELL, wrap={R: 1}, content={A: 1}, W=True, Y=True)]),
        _r(TOP, 0.05 * s, comp=_pat(CELL, wrap={R: 1}),                          # 5 receptor turnover
           comps=[_ctor(CELL, W=True, Y=True)]),
        _r(TOP, 0.0004 * s, comp=_pat(CELL, content={A: 2}),                     # 6 division
           comps=[_ctor(CELL, content={A: 1}, W=True, Y=True), _ctor(CELL, wrap={R: 2}, content={A: 1})]),
        _r(TOP, 0.03 * s, comp=_pat(CELL), release_W=True, release_Y=True),      # 7 lysis
        _r(CELL, 0.0002 * s, atoms={A: 2}, comps=[_ctor(VES, content={B: 1})]),  # 8 vesicle formation
        _r(CELL, 0.05 * s, comp=_pat(VES), release_Y=True),                      # 9 fusion (W dropped)
        _r(VES, 0.2 * s, atoms={A: 1}, rhs_atoms={B: 1}),                        # 10 loading (never: no a in VES)
        _r(CELL, 0.1 * s, atoms={B: 1}, rhs_atoms={P: 1}),                       # 11 cargo processing
        _r(TOP, 0.5 * s, comp=_pat(CELL, content={P: 1}), rhs_atoms={P: 1},      # 12 export
           comps=[_ctor(CELL, W=True, Y=True)]),
        _r(TOP, 0.2 * s, atoms={A: 1}),                                          # 13 decay of released a
        _r(TOP, 0.2 * s, atoms={R: 1}),                                          # 14 ... r
        _r(TOP, 0.2 * s, atoms={B: 1}),                                          # 15 ... b
        _r(TOP, 0.1 * s, atoms={P: 1}),                                          # 16 ... p
        _r(TOP, 0.1 * s, comp=_pat(VES)),                                        # 17 free vesicles decay (deleted)
        _r(VES, 0.001 * s, atoms={B: 2}, X=False, rhs_atoms={P: 1}),             # 18 vesicle collapse (no X)
        _r(CELL, 1e-5 * s, atoms={P: 2}, X=False, rhs_atoms={A: 2}),             # 19 clear-out (no X)
        _r(CELL, 0.1 * s, atoms={A: 1}),                                         # 20 decay of a in cells
    ]
    cells = [{"label": CELL, "wrap": {R: r0}, "content": {"atoms": {A: a0}}} for _ in range(n_cells)]
    term = {"atoms": {N: n0}, "comps": cells}
    observables = [("count", CELL), ("count", VES), ("content", TOP, N), ("content", CELL, A),
                   ("wrap", CELL, R), ("content", VES, B), [("content", TOP, P), ("content", CELL, P)],
                   ("content", CELL, N)]
    return {"name": "cell population", "n_atoms": 5, "n_labels": 3, "term": term, "rules": rules,
            "observables": observables}


def random_dynamic_model(seed, n_atoms=4, n_labels=3, n_rules=14, depth=2):
    """Random small dynamic models for parity cases: rule shapes drawn
    uniformly from the calculus's (local / child-pattern, X kept or not,
    release of W / Y, in-place and appended constructors), reaction order
    <= 2 over context + wrap + content atoms, rates 10^U(-2, 0.5).  The
    initial term nests compartments up to `depth` levels below TOP."""
    rnd = random.Random(seed)

    def ms(k):
        out = {}
        for _ in range(k):
            a = rnd.randrange(n_atoms)
            out[a] = out.get(a, 0) + 1
        return out

    def term(level):
        t = {"atoms": {a: rnd.randint(0, 12) for a in range(n_atoms)}, "comps": []}
        if level < depth:
            for _ in range(rnd.randint(0, 3)):
                t["comps"].append({"label": rnd.randrange(1, n_labels), "wrap": {a: rnd.randint(0, 4) for a in range(n_atoms)},
                                   "content": term(level + 1)})
        return t

    rules = []
    for _ in range(n_rules):
        label = rnd.randrange(n_labels)
        rate = 10.0 ** rnd.uniform(-2.0, 0.5)
        if rnd.random() < 0.45:
            order = rnd.randint(0, 2)
            rules.append(_r(label, rate, atoms=ms(order), X=rnd.random() > 0.1, rhs_atoms=ms(rnd.randint(0, 2)),
                            comps=[_ctor(rnd.randrange(1, n_labels), wrap=ms(rnd.randint(0, 1)), content=ms(rnd.randint(0, 2)))]
                            if rnd.random() < 0.15 else []))
            continue
        order = rnd.randint(0, 2)
        where = [rnd.randrange(3) for _ in range(order)]
        ctx, wr, ct = {}, {}, {}
        for wh in where:
            d = (ctx, wr, ct)[wh]
            a = rnd.randrange(n_atoms)
            d[a] = d.get(a, 0) + 1
        clab = rnd.randrange(1, n_labels)
        shape = rnd.randrange(5)
        rel_w = rel_y = False
        comps = []
        if shape == 0:    # in-place rewrite (transport-like)
            comps = [_ctor(rnd.randrange(1, n_labels), wrap=ms(rnd.randint(0, 1)), content=ms(rnd.randint(0, 2)), W=True, Y=True)]
        elif shape == 1:  # dissolution
            rel_w, rel_y = rnd.random() < 0.7, True
        elif shape == 2:  # deletion of the child
            pass
        elif shape == 3:  # division-like: in place + appended
            comps = [_ctor(clab, content=ms(rnd.randint(0, 1)), W=True, Y=True),
                     _ctor(clab, wrap=ms(rnd.randint(0, 1)), content=ms(rnd.randint(0, 2)))]
        else:             # W and Y moved into new, appended compartments
            comps = [_ctor(rnd.randrange(1, n_labels), content=ms(1), Y=True), _ctor(clab, W=True)]
        rules.append(_r(label, rate, atoms=ctx, comp=_pat(clab, wrap=wr, content=ct), X=rnd.random() > 0.1,
                        rhs_atoms=ms(rnd.randint(0, 2)), release_W=rel_w, release_Y=rel_y, comps=comps))
    observables = [("count", l) for l in range(1, n_labels)] + \
                  [("content", l, a) for l in range(n_labels) for a in range(n_atoms)] + \
                  [("wrap", l, a) for l in range(1, n_labels) for a in range(min(2, n_atoms))]
    return {"name": "random dynamic %d" % seed, "n_atoms": n_atoms, "n_labels": n_labels, "term": term(0),
            "rules": rules, "observables": observables}


CONFIG_C6 = dict(desc="dynamic CWC cell population", t_end=20.0, sample_dt=0.1, n_replicas=8192, seed=1)
