"""Pins for the oracle's simulation loop against closed forms, the chemical
master equation, invariants and the sampling / termination conventions.

Closed forms (BASELINE north_star; SURVEY §8(c) "What pins each part"):
  immigration-death from 0: X(t) ~ Poisson(100 (1 - e^{-0.1 t})) at every t;
  pure decay: Binomial(N0, e^{-kt});
  isomerisation A <-> B: A(t) ~ Binomial(N, p(t));
  any first-order network: E[x(t)] solves the linear ODE (expm).
CME brute force: A+A->D, tiny Michaelis-Menten (tests/cme.py).
"""
import math

import numpy as np
import pytest
from scipy.linalg import expm
from scipy.stats import binom, poisson

import oracle
import workloads as w

from .cme import chi2_pvalue, solve

Z = 4.5  # |z| bound; with Bonferroni over the tested cells the family p is ~1e-3


def _mean_var(res, o=0):
    cnt = res["count"][0, :, o].astype(float)
    s1 = res["sum"][0, :, o].astype(float)
    s2 = np.array([oracle.moments.sumsq_int(q) for q in res["sumsq"][0, :, o]], dtype=float)
    mean = s1 / cnt
    var = (s2 - cnt * mean**2) / (cnt - 1)
    return mean, var


def test_decay_mean_at_t1_spec():
    # S:241 / S:512: 1000 instances of a -> 0 (k=1) from 1000: mean at t=1 within 3 s.e. of 367.879
    res = oracle.simulate(w.decay_model(1000, 1.0), 1000, 1.0, 0.5, seed=1, want_traj=True)
    x1 = res["traj"][:, 2, 0]
    se = x1.std(ddof=1) / math.sqrt(len(x1))
    assert abs(x1.mean() - 1000 * math.exp(-1)) < 3 * se
    p = math.exp(-1)
    assert abs(x1.var(ddof=1) - 1000 * p * (1 - p)) < 5 * 1000 * p * (1 - p) * math.sqrt(2 / 999)


def test_immigration_death_poisson_every_sample():
    d, _, cfg = w.config("C1")
    res = oracle.simulate(d, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
    n = cfg["n_replicas"]
    t = np.arange(101) * 1.0
    m = 100.0 * (1.0 - np.exp(-0.1 * t))
    mean, var = _mean_var(res)
    assert mean[0] == 0 and var[0] == 0
    z = (mean[1:] - m[1:]) / np.sqrt(m[1:] / n)
    assert np.abs(z).max() < Z
    # Poisson: variance equals the mean (check at t >= 10 with the var-of-var bound)
    for j in (10, 30, 60, 100):
        sd = math.sqrt(2 * m[j] ** 2 / (n - 1) + m[j] / n)
        assert abs(var[j] - m[j]) < Z * sd
    # full pmf at t = 50 and t = 100
    for j in (50, 100):
        vals = res["traj"][:, j, 0]
        ks = np.arange(0, 250)
        obs = np.bincount(vals, minlength=250)[:250]
        assert chi2_pvalue(obs, poisson.pmf(ks, m[j]), n) > 1e-4
    # E[firings] = k_in T + k_out int_0^T m = 1900.0045
    assert abs(res["firings"].mean() - 1900.0045) < 0.01 * 1900
    assert (res["status"] == oracle.ST_DONE).all()


def test_isomerisation_binomial():
    N, kf, kb = 20, 1.0, 0.5
    d = w.isomerisation_model(N, kf, kb)
    n = 4000
    res = oracle.simulate(d, n, 3.0, 0.25, seed=11)
    for j in (2, 4, 12):
        t = 0.25 * j
        p = kb / (kf + kb) + kf / (kf + kb) * math.exp(-(kf + kb) * t)
        a = res["traj"][:, j, 0]
        assert ((a + res["traj"][:, j, 1]) == N).all()
        obs = np.bincount(a, minlength=N + 1)
        assert chi2_pvalue(obs, binom.pmf(np.arange(N + 1), N, p), n) > 1e-4


def test_cme_dimerisation():
    d = w.dimerisation_model(6, 1.0)
    times = [0.25, 0.5, 1.0]
    states, ps = solve(d, times)
    n = 20000
    res = oracle.simulate(d, n, 1.0, 0.25, seed=3)
    # C(n,2) vs n(n-1) convention separates here: E[A](0.5) = 1.6928
    ea = sum(p * s[0] for p, s in zip(ps[1], states))
    assert abs(ea - 1.6928) < 1e-3
    for t, p in zip(times, ps):
        j = int(round(t / 0.25))
        idx = {s: i for i, s in enumerate(states)}
        obs = np.zeros(len(states))
        for row in res["traj"][:, j, :]:
            obs[idx[tuple(int(v) for v in row)]] += 1
        assert chi2_pvalue(obs, p, n) > 1e-4


def test_cme_michaelis_menten_tiny():
    d = w.michaelis_menten_model(kf=1.0, kr=1.0, kcat=1.0, e0=2, s0=4)
    times = [0.5, 1.0, 2.0]
    states, ps = solve(d, times)
    n = 20000
    res = oracle.simulate(d, n, 2.0, 0.5, seed=5)
    idx = {s: i for i, s in enumerate(states)}
    for t, p in zip(times, ps):
        j = int(round(t / 0.5))
        obs = np.zeros(len(states))
        for row in res["traj"][:, j, :]:
            obs[idx[tuple(int(v) for v in row)]] += 1
        assert chi2_pvalue(obs, p, n) > 1e-4


def _linear_compartment_model():
    """First-order compartment network: every rule has order <= 1."""
    R = w.models._rule
    return {
        "name": "linear_cwc", "n_types": 2, "n_species": 2,
        "parent": [-1, 0, 0, 0], "type": [0, 1, 1, 1],
        "rules": [R(0, [], [(0, 0, 1)], 20.0), R(0, [(0, 0, 1)], [], 0.2),
                  R(1, [(0, 0, 1)], [(0, 1, 1)], 0.7), R(1, [(0, 1, 1)], [], 0.3),
                  R(0, [(0, 0, 1)], [(1, 0, 1)], 0.1, child_label=1),
                  R(0, [(1, 1, 1)], [(0, 1, 1)], 0.4, child_label=1)],
        "init": [30, 0, 5, 0, 0, 7, 2, 2],
        "n_obs": 8, "obs_of_cell": list(range(8)),
    }


def _linear_mean_ode(d):
    """The test's own reading of the mass-action mean ODE of a model whose
    rules all have order <= 1: dE[x]/dt = A E[x] + b (each rule applied in
    every context of its label, and for every matching child)."""
    S = int(d["n_species"])
    C = len(d["parent"])
    nc = S * C
    A = np.zeros((nc, nc))
    b = np.zeros(nc)
    for r in d["rules"]:
        for c in range(C):
            if d["type"][c] != r["label"]:
                continue
            kids = [None] if r["child_label"] < 0 else [q for q in range(C) if d["parent"][q] == c and d["type"][q] == r["child_label"]]
            for q in kids:
                cell = lambda wh, s: (c if wh == 0 else q) * S + s  # noqa: E731
                nu = np.zeros(nc)
                for (wh, s, m) in r["products"]:
                    nu[cell(wh, s)] += m
                src = None
                for (wh, s, m) in r["reactants"]:
                    assert m == 1 and src is None, "order <= 1 only"
                    nu[cell(wh, s)] -= m
                    src = cell(wh, s)
                if src is None:
                    b += r["rate"] * nu
                else:
                    A[:, src] += r["rate"] * nu
    return A, b


def _check_linear_mean(d, n, t_end, dt, seed, samples, cells=None):
    A, b = _linear_mean_ode(d)
    nc = A.shape[0]
    aug = np.zeros((nc + 1, nc + 1))
    aug[:nc, :nc] = A
    aug[:nc, nc] = b
    res = oracle.simulate(d, n, t_end, dt, seed=seed)
    x0 = np.array(list(d["init"]) + [1], dtype=float)
    # observables are sums of cells: map the cell means through obs_of_cell
    O = int(d["n_obs"])
    Mo = np.zeros((O, nc))
    for cidx, o in enumerate(d["obs_of_cell"]):
        if o >= 0:
            Mo[o, cidx] = 1.0
    for j in samples:
        m = Mo @ (expm(aug * (j * dt)) @ x0)[:nc]
        vals = res["traj"][:, j, :].astype(float)
        # standard error, floored at one event in n trajectories (observables
        # with very small rates may see no event at all in the sample)
        se = np.maximum(vals.std(axis=0, ddof=1), 1.0) / math.sqrt(n)
        z = (vals.mean(axis=0) - m) / se
        assert np.abs(z).max() < Z, (j, z)


def test_first_order_network_mean_matches_linear_ode():
    _check_linear_mean(_linear_compartment_model(), 3000, 4.0, 1.0, 2, (1, 2, 4))


def test_c5_structure_linearised_mean_matches_linear_ode():
    """The C5 CWC model (33 compartments, transport through child patterns)
    with its dimerisation rules removed is first order: its mean obeys the
    linear ODE exactly.  Pins the oracle's flattening of the real C5 tree
    (1172 -> 1044 flat reactions), rates and per-type observables."""
    d = dict(w.config("C5")[0])
    d["rules"] = [r for r in d["rules"] if sum(m for (_, _, m) in r["reactants"]) <= 1]
    assert len(d["rules"]) == 56 - 8
    _check_linear_mean(d, 160, 0.2, 0.05, 3, (1, 2, 4))


def test_c4_first_order_subnetwork_mean_matches_linear_ode():
    """The C4 random network restricted to its order-0/1 reactions: mean vs the
    linear ODE (pins propensities k*x and k for the generated rules)."""
    d = dict(w.config("C4")[0])
    d["rules"] = [r for r in d["rules"] if sum(m for (_, _, m) in r["reactants"]) <= 1]
    assert 100 < len(d["rules"]) < 256
    _check_linear_mean(d, 300, 0.2, 0.05, 4, (1, 2, 4))


def test_mm_conservation_every_sample():
    d, sweep, cfg = w.config("C3")
    g = list(range(0, 4096 * 16, 331))
    res = oracle.simulate(d, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                          g_list=g, want_stats=False)
    tr = res["traj"]
    assert ((tr[:, :, 0] + tr[:, :, 2]) == 200).all()
    assert ((tr[:, :, 1] + tr[:, :, 2] + tr[:, :, 3]) == 1000).all()
    assert (tr >= 0).all()


def test_samples_are_pre_event_piecewise_constant_state():
    """Reconstruct each trajectory from its trace (event times tn, chosen mu)
    and check sample j equals the state after all events with tn < j*dt
    (pre-event at ties), that exactly J+1 samples exist
    and that sample 0 is x0."""
    d = w.lotka_volterra_model(k1=1.0, k2=0.005, k3=1.0, x0=40, y0=40)
    fm = oracle.FlatModel(d)
    dt, t_end = 0.05, 3.0
    for g in range(6):
        res = oracle.simulate(d, 8, t_end, dt, seed=9, g_list=[g], trace_g=g, trace_cap=100000, flat=fm)
        tr = res["trace"]
        traj = res["traj"][0]
        assert traj.shape[0] == int(math.floor(t_end / dt)) + 1
        assert tr[-1][4] == -1.0 and (tr[:-1, 4] >= 0).all()
        assert res["firings"][0] == len(tr) - 1
        # counter n increments by one per drawn block
        assert (tr[:, 0] == np.arange(len(tr))).all()
        x = np.array(d["init"], dtype=np.int64)
        ev = 0
        t_prev = 0.0
        for j in range(traj.shape[0]):
            tj = j * dt
            while ev < len(tr) - 1 and tr[ev][3] < tj:
                assert tr[ev][3] == t_prev + tr[ev][2]
                t_prev = tr[ev][3]
                for (c, dd) in fm.entries[int(tr[ev][4])]["nu"]:
                    x[c] += dd
                ev += 1
            assert (traj[j] == x).all(), (g, j)


def test_stall_fills_remaining_samples():
    d = w.decay_model(3, 5.0)
    res = oracle.simulate(d, 50, 10.0, 1.0, seed=4)
    assert (res["status"] == oracle.ST_STALLED).all()
    assert (res["firings"] == 3).all()
    assert (res["traj"][:, -3:, 0] == 0).all()
    assert (res["count"] == 50).all()


def test_overflow_freezes_state():
    d = w.immigration_death_model(k_in=1e6, k_out=1e-12, a0=2**31 - 5)
    res = oracle.simulate(d, 4, 1.0, 0.5, seed=1)
    assert (res["status"] == oracle.ST_OVERFLOW).all()
    assert (res["firings"] == 4).all()
    assert (res["traj"][:, -1, 0] == 2**31 - 1).all()


def test_finalize_spec_examples():
    # [1,2,3] -> mean 2, var 1 ; single value -> var 0 ; ci90(var=4, n=100) = 0.32898
    m, v, c = oracle.moments.finalize_cell(3, 6, 14)
    assert (m, v) == (2.0, 1.0)
    assert oracle.moments.finalize_cell(1, 7, 49) == (7.0, 0.0, 0.0)
    assert abs(1.6449 * math.sqrt(4 / 100) - 0.32898) < 1e-5
    n, s1 = 100, 0
    # a set with var 4 exactly: 50 values of -2+10 and 50 of 2+10 -> var = 400/99
    vals = [8] * 50 + [12] * 50
    m, v, c = oracle.moments.finalize_cell(len(vals), sum(vals), sum(x * x for x in vals))
    assert m == 10.0 and abs(v - 400 / 99) < 1e-12
    assert abs(c - 1.6449 * math.sqrt(v / 100)) < 1e-12


def test_finalize_matches_two_pass_on_oracle_trajectories():
    d, _, cfg = w.config("C1")
    res = oracle.simulate(d, 256, cfg["t_end"], cfg["sample_dt"], 1)
    means, vars_, _ = oracle.finalize(res["count"], res["sum"], res["sumsq"])
    x = res["traj"][:, :, 0].astype(float)
    tp_mean = x.mean(axis=0)
    tp_var = x.var(axis=0, ddof=1)
    assert np.allclose(means, tp_mean, rtol=1e-12, atol=0)
    assert np.allclose(vars_, tp_var, rtol=1e-9, atol=1e-12)
    assert (res["count"] == 256).all()


def test_statistics_equal_host_reduction_of_trajectories():
    d, sweep, cfg = w.config("C3")
    g = list(range(0, 64 * 16))  # first 64 points, all replicas
    res = oracle.simulate(d, 16, cfg["t_end"], cfg["sample_dt"], 1, sweep=sweep, g_list=g)
    tr = res["traj"].reshape(64, 16, -1, 4)
    assert (res["count"][:64] == 16).all()
    assert (res["sum"][:64] == tr.sum(axis=1)).all()
    sq = (tr.astype(object) ** 2).sum(axis=1)
    got = np.vectorize(lambda lo, hi: int(lo) | (int(hi) << 64), otypes=[object])(
        res["sumsq"][:64, ..., 0], res["sumsq"][:64, ..., 1])
    assert (got == sq).all()


@pytest.mark.parametrize("cfgname", ["C1", "C2", "C3", "C4", "C5"])
def test_sample_grid_is_exact(cfgname):
    cfg = w.CONFIGS[cfgname]
    J = math.floor(cfg["t_end"] / cfg["sample_dt"])
    assert J * cfg["sample_dt"] == cfg["t_end"]
    assert oracle.n_samples(cfg["t_end"], cfg["sample_dt"]) == J + 1
