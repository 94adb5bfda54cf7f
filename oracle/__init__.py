"""CPU oracle of the bulk direct-method SSA hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package.  It shares no code with `paper_1010_2438_b200/` (the product path):
its own flattening (`flatten.py`), its own Philox, propensities, sampling loop
and exact-integer statistics (`ssa_oracle.c`), its own finalize (`moments.py`).
The only shared input is `workloads/` (model descriptions, no arithmetic).

Parity status of each function:
  flatten            pinned: paper example P:193-196, brute-force enumeration
  philox4x32_10      pinned: at::philox_engine (torch header, compiled in tests)
  uniforms / tau     pinned: closed-form bit patterns, S:203-205
  binomial           pinned: math.comb
  simulate           pinned: closed forms (decay, immigration-death,
                     isomerisation, first-order mean ODE), CME brute force
                     (scipy expm), conservation invariants
  finalize           pinned: S:418-427 worked values, two-pass statistics
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .flatten import flatten  # noqa: F401
from .moments import finalize  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ssa_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

ST_DONE, ST_STALLED, ST_OVERFLOW = 0, 1, 2


def build(force=False):
    """Compile the C oracle (gcc -O2 -ffp-contract=off, glibc libm)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Model(ctypes.Structure):
    _fields_ = [("n_cells", ctypes.c_int32), ("n_reactions", ctypes.c_int32), ("n_obs", ctypes.c_int32)] + [
        (n, ctypes.c_void_p) for n in ("re_ptr", "re_cell", "re_mult", "nu_ptr", "nu_cell", "nu_delta",
                                       "rule_of", "init", "obs_of_cell")]


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        _lib.oracle_simulate.restype = ctypes.c_int
        _lib.oracle_simulate.argtypes = [P, ctypes.c_int32, P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_int64,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                         P, P, P, P, P, P, ctypes.c_int64, P, ctypes.c_int64, P]
        _lib.oracle_philox4x32_10.argtypes = [P, P, P]
        _lib.oracle_uniforms.argtypes = [P, P, P]
        _lib.oracle_propensities.argtypes = [P, P, P, P]
        _lib.oracle_select.restype = ctypes.c_int
        _lib.oracle_select.argtypes = [P, ctypes.c_int, ctypes.c_double]
        _lib.oracle_tau_stream.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                           ctypes.c_double, P, P]
        _lib.oracle_tau.restype = ctypes.c_double
        _lib.oracle_tau.argtypes = [ctypes.c_double, ctypes.c_double]
        _lib.oracle_binomial.restype = ctypes.c_int64
        _lib.oracle_binomial.argtypes = [ctypes.c_int64, ctypes.c_int64]
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def philox4x32_10(ctr, key):
    lib = _load()
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib.oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return [int(v) for v in out]


def uniforms(w):
    lib = _load()
    ww = np.asarray(w, dtype=np.uint32)
    u1 = ctypes.c_double()
    u2 = ctypes.c_double()
    lib.oracle_uniforms(_ptr(ww), ctypes.byref(u1), ctypes.byref(u2))
    return u1.value, u2.value


def tau(u1, a0):
    """The oracle's time step tau = (-log u1) / a0 (the function its loop calls)."""
    return float(_load().oracle_tau(float(u1), float(a0)))


def tau_stream(seed, g, n0, count, a0):
    """(tau, u2) arrays the oracle draws for firings n0.. of trajectory g at total rate a0."""
    lib = _load()
    tau = np.zeros(count, dtype=np.float64)
    u2 = np.zeros(count, dtype=np.float64)
    lib.oracle_tau_stream(seed, g, n0, count, float(a0), _ptr(tau), _ptr(u2))
    return tau, u2


def binomial(n, k):
    return int(_load().oracle_binomial(n, k))


class FlatModel:
    """Oracle-side flat tables (from oracle.flatten) as contiguous arrays."""

    def __init__(self, desc):
        self.desc = desc
        self.entries = flatten(desc)
        S = int(desc["n_species"])
        C = len(desc["parent"])
        self.n_cells = S * C
        self.M = len(self.entries)
        self.n_rules = len(desc["rules"])
        self.n_obs = int(desc["n_obs"])
        re_ptr, re_cell, re_mult, nu_ptr, nu_cell, nu_delta = [0], [], [], [0], [], []
        for e in self.entries:
            for (c, k) in e["reactants"]:
                re_cell.append(c)
                re_mult.append(k)
            re_ptr.append(len(re_cell))
            for (c, d) in e["nu"]:
                nu_cell.append(c)
                nu_delta.append(d)
            nu_ptr.append(len(nu_cell))
        i32 = lambda v: np.ascontiguousarray(np.asarray(v if len(v) else [0], dtype=np.int32))  # noqa: E731
        self._arrays = dict(
            re_ptr=i32(re_ptr), re_cell=i32(re_cell), re_mult=i32(re_mult),
            nu_ptr=i32(nu_ptr), nu_cell=i32(nu_cell), nu_delta=i32(nu_delta),
            rule_of=i32([e["rule"] for e in self.entries]),
            init=i32(desc["init"]), obs_of_cell=i32(desc["obs_of_cell"]))
        self._c = _Model(self.n_cells, self.M, self.n_obs,
                         *[self._arrays[n].ctypes.data for n in ("re_ptr", "re_cell", "re_mult", "nu_ptr", "nu_cell",
                                                                 "nu_delta", "rule_of", "init", "obs_of_cell")])

    def rule_rates(self, sweep=None):
        base = [float(r["rate"]) for r in self.desc["rules"]]
        if sweep is None:
            return np.asarray([base], dtype=np.float64)
        rows = []
        for vals in sweep["values"]:
            row = list(base)
            for rid, v in zip(sweep["rules"], vals):
                row[rid] = float(v)
            rows.append(row)
        return np.ascontiguousarray(np.asarray(rows, dtype=np.float64))


def propensities(fm, x, rule_rates_row=None):
    """Oracle propensities a[m] for state x (length n_cells) with the model's
    own rates (or one row of FlatModel.rule_rates)."""
    lib = _load()
    rates = fm.rule_rates()[0] if rule_rates_row is None else np.asarray(rule_rates_row, dtype=np.float64)
    k = np.ascontiguousarray(np.asarray([rates[e["rule"]] for e in fm.entries] or [0.0], dtype=np.float64))
    xx = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    a = np.zeros(max(fm.M, 1), dtype=np.float64)
    lib.oracle_propensities(ctypes.byref(fm._c), _ptr(k), _ptr(xx), _ptr(a))
    return a[: fm.M]


def select(a, target):
    lib = _load()
    aa = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return int(lib.oracle_select(_ptr(aa), len(aa), float(target)))


def n_samples(t_end, dt):
    return int(np.floor(t_end / dt)) + 1


def simulate(desc, n_replicas, t_end, sample_dt, seed, sweep=None, g_list=None,
             want_traj=True, want_stats=True, trace_g=-1, trace_cap=0, flat=None):
    """Run the oracle on trajectories g_list (default: all).  Returns a dict:
    traj [n_g][J+1][O] int64, firings [n_g], status [n_g],
    count/sum [P][J+1][O] int64, sumsq [P][J+1][O] as python-int-exact
    uint64 (lo, hi) pairs, trace [n][5]."""
    lib = _load()
    fm = flat or FlatModel(desc)
    rates = fm.rule_rates(sweep)
    P = rates.shape[0]
    G = P * n_replicas
    g = np.arange(G, dtype=np.int64) if g_list is None else np.ascontiguousarray(np.asarray(g_list, dtype=np.int64))
    J1 = n_samples(t_end, sample_dt)
    O = fm.n_obs
    traj = np.zeros((len(g), J1, O), dtype=np.int64) if want_traj else None
    firings = np.zeros(len(g), dtype=np.int64)
    status = np.zeros(len(g), dtype=np.int32)
    if want_stats:
        cnt = np.zeros((P, J1, O), dtype=np.int64)
        sm = np.zeros((P, J1, O), dtype=np.int64)
        sq = np.zeros((P, J1, O, 2), dtype=np.uint64)
    else:
        cnt = sm = sq = None
    trace = np.zeros((max(trace_cap, 1), 5), dtype=np.float64)
    trace_n = ctypes.c_int64(0)
    rc = lib.oracle_simulate(ctypes.byref(fm._c), fm.n_rules, _ptr(rates), P, n_replicas, _ptr(g), len(g),
                             float(t_end), float(sample_dt), int(seed),
                             _ptr(traj), _ptr(firings), _ptr(status), _ptr(cnt), _ptr(sm), _ptr(sq),
                             int(trace_g), _ptr(trace) if trace_cap > 0 else None, int(trace_cap),
                             ctypes.byref(trace_n))
    if rc != 0:
        raise ValueError("oracle_simulate: invalid arguments")
    return dict(traj=traj, firings=firings, status=status, count=cnt, sum=sm, sumsq=sq,
                trace=trace[: trace_n.value], g=g, n_points=P, J1=J1)
