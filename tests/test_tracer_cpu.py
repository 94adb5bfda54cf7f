"""CPU tests of the divergence tracer (tests/tracer.py) on oracle traces: the
state rebuild is pinned against the oracle's own a0 at every record, and the
classification accepts only verified ulp-level causes (a perturbed a0 or mu
beyond the summation error bound, an unexplained tau difference, identical
traces under a sample mismatch, or a sample mismatch before the first
differing firing are all BUG)."""
import math

import numpy as np
import pytest

import oracle
import workloads as w

from .tracer import KernelGeom, OracleSide, classify, first_sample_mismatch_t, gamma


def _oracle_trace(desc, cfg, g, cap=100000):
    r = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], g_list=[g],
                        want_stats=False, trace_g=g, trace_cap=cap)
    return [tuple(x) for x in r["trace"]], r["traj"][0]


def _next_up(x, k=1):
    for _ in range(k):
        x = math.nextafter(x, math.inf)
    return x


CASES = [("lv4", lambda: w.lotka_volterra_chain(4), dict(t_end=0.05, sample_dt=0.01, n_replicas=4, seed=3)),
         ("rnd24", lambda: w.random_network_model(seed=5, n_species=8, n_reactions=24),
          dict(t_end=0.05, sample_dt=0.01, n_replicas=4, seed=2)),
         ("cwc", lambda: w.small_cwc_model(3, 1), dict(t_end=3.0, sample_dt=0.5, n_replicas=4, seed=1))]


@pytest.mark.parametrize("name,make,cfg", CASES, ids=[c[0] for c in CASES])
def test_state_rebuild_reproduces_oracle_a0_at_every_record(name, make, cfg):
    desc = make()
    tr, _ = _oracle_trace(desc, cfg, 2)
    side = OracleSide(desc, None, cfg["n_replicas"], cfg["seed"])
    assert len(tr) > 20
    x = side.x0.copy()
    for i, rec in enumerate(tr):
        a = side.propensities(2, x)
        s = 0.0
        for k, v in enumerate(a):
            s = v if k == 0 else s + float(v)
        assert s == rec[1], i
        if rec[4] >= 0:
            for c, d in side.nu[int(rec[4])]:
                x[c] += d


def test_classification_is_verified():
    desc = w.random_network_model(seed=5, n_species=8, n_reactions=24)
    cfg = dict(t_end=0.05, sample_dt=0.01, n_replicas=4, seed=2)
    g = 1
    tr, traj = _oracle_trace(desc, cfg, g)
    side = OracleSide(desc, None, cfg["n_replicas"], cfg["seed"])
    M = len(side.fm.entries)
    warp, thread = KernelGeom(True, 16, M), KernelGeom(False, M=M)
    i = len(tr) // 2
    # identical traces: fine only if the samples agree
    assert classify(tr, tr, warp, side, g)[0] == "identical-trace"
    assert classify(tr, tr, warp, side, g, sample_mismatch_t=0.03)[0] == "BUG"
    # a0 one ulp off (the GPU's t' consistent with it): a sum-order difference on a warp kernel only
    rec = tr[i]
    t_prev = tr[i - 1][3]
    a0 = _next_up(rec[1])
    gpu = list(tr)
    gpu[i] = (rec[0], a0, rec[2], t_prev + rec[2], rec[4])
    assert classify(gpu, tr, warp, side, g)[0] == "a0-sum-order"
    assert classify(gpu, tr, thread, side, g)[0] == "BUG"
    # far beyond the summation bound
    gpu[i] = (rec[0], rec[1] * (1 + 1e-9), rec[2], t_prev + rec[2], rec[4])
    assert classify(gpu, tr, warp, side, g)[0] == "BUG"
    # tau one ulp off: log-ulp only if the device E explains it exactly
    u1, _ = side.uniforms(g, int(rec[0]))
    E_ora = oracle.tau(u1, 1.0)
    E_alt = _next_up(E_ora)
    tau_alt = E_alt / rec[1]
    gpu[i] = (rec[0], rec[1], tau_alt, t_prev + tau_alt, rec[4])
    cat = classify(gpu, tr, warp, side, g, draw_E=lambda gg, n: E_alt)[0]
    exact_ok = abs(E_alt - (-math.log(u1))) <= math.ulp(E_ora)
    assert cat == ("log-ulp" if exact_ok and tau_alt != rec[2] else "BUG")
    assert classify(gpu, tr, warp, side, g, draw_E=lambda gg, n: E_ora)[0] == "BUG"
    # t' inconsistent with t + tau
    gpu[i] = (rec[0], rec[1], rec[2], _next_up(rec[3], 3), rec[4])
    assert classify(gpu, tr, warp, side, g)[0] == "BUG"
    # a different mu far from any prefix boundary: BUG even on a warp kernel
    mu = int(rec[4])
    gpu[i] = (rec[0], rec[1], rec[2], rec[3], float((mu + 5) % M))
    assert classify(gpu, tr, warp, side, g)[0] == "BUG"
    # the first sample mismatch must not precede the divergence
    gpu[i] = (rec[0], _next_up(rec[1]), rec[2], t_prev + rec[2], rec[4])
    assert classify(gpu, tr, warp, side, g, sample_mismatch_t=0.0)[0] == "BUG"
    assert classify(gpu, tr, warp, side, g, sample_mismatch_t=rec[3] + 1e-6)[0] == "a0-sum-order"


def test_first_sample_mismatch_and_gamma():
    a = np.zeros((5, 3), dtype=np.int64)
    b = a.copy()
    assert first_sample_mismatch_t(a, b, 0.5) is None
    b[3, 1] = 7
    assert first_sample_mismatch_t(a, b, 0.5) == 1.5
    assert gamma(0) == 0.0 and 10 * 2.0**-53 < gamma(10) < 10.001 * 2.0**-53
