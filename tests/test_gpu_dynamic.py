"""GPU parity of the dynamic-topology path (include/cwc_dyn.h, SURVEY 8(f)
NEXT-4) against the dynamic CPU oracle oracle/dynamic.py (pinned in
tests/test_oracle_dynamic_topology.py):

  * the C6 cell-population workload (creation, division, lysis releasing
    nested vesicles, fusion, deletion, rules without X) at its full horizon
    and sampling step, and 17 random models whose rule shapes are drawn from
    the whole calculus (in-place rewrites, dissolution with W / Y, deletion,
    division, W and Y moved into appended compartments, no-X rules at every
    label, nested initial terms up to depth 2);
  * bar: every sampled observable, firing count and status equal to the
    oracle's for every compared trajectory (the device sums a0 in a
    different order -- DESIGN.md section 4's warp-path class -- so a
    divergence is possible in principle at ~1e-9 per trajectory; none is
    accepted here), and the on-line moments equal the exact reduction of the
    oracle trajectories;
  * launch-shape invariance (warps per CTA, CTAs per SM), sharding by
    replica offset, and the CAPACITY status of a term that outgrows the
    device capacity (samples before the overflowing creation equal the
    oracle's; the rest hold the frozen term).
"""
import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import workloads.dynamic as wd  # noqa: E402
from oracle import dynamic as dyn  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1010_2438_b200 import cwc_dyn  # noqa: E402

RANDOM_SEEDS = [0, 2, 3, 5, 7, 9, 12, 13, 17, 18, 20, 21, 25, 28, 32, 35, 38]


def _model(spec):
    kind, arg = spec
    if kind == "cell":
        return wd.cell_population_model(**arg)
    if kind == "random":
        return wd.random_dynamic_model(arg)
    if kind == "creation":
        return creation_model()
    raise KeyError(kind)


def _oracle_chunk(args):
    spec, t_end, dt, seed, g_chunk = args
    r = dyn.simulate(_model(spec), 0, t_end, dt, seed, g_list=g_chunk)
    return r["traj"], r["firings"], r["status"]


def oracle_runs(spec, t_end, dt, seed, g_list):
    workers = max(1, min(os.cpu_count() or 1, 32))
    n_chunks = max(1, min(len(g_list), 4 * workers))
    chunks = [g_list[i::n_chunks] for i in range(n_chunks)]
    with cf.ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_oracle_chunk, [(spec, t_end, dt, seed, c) for c in chunks]))
    J1, O = res[0][0].shape[1:]
    traj = np.zeros((len(g_list), J1, O), dtype=np.int64)
    fir = np.zeros(len(g_list), dtype=np.int64)
    st = np.zeros(len(g_list), dtype=np.int32)
    for i, (t, f, s) in enumerate(res):
        traj[i::n_chunks] = t
        fir[i::n_chunks] = f
        st[i::n_chunks] = s
    return traj, fir, st


def creation_model():
    """Compartments created at a constant rate and never removed (the count
    only grows): exercises the CAPACITY status."""
    return {"name": "creation", "n_atoms": 1, "n_labels": 2, "term": {"atoms": {0: 5}, "comps": []},
            "rules": [{"label": 0, "atoms": {}, "rate": 2.0,
                       "rhs": {"X": True, "atoms": {}, "comps": [{"label": 1, "wrap": {}, "content": {0: 1}}]}},
                      {"label": 1, "atoms": {0: 1}, "rate": 0.5, "rhs": {"X": True, "atoms": {0: 2}}}],
            "observables": [("count", 1), ("content", 1, 0), ("content", 0, 0)]}


def _moments(traj):
    t = traj.astype(object)
    return (np.full(traj.shape[1:], traj.shape[0], dtype=np.int64), t.sum(axis=0), (t * t).sum(axis=0))


def _check(spec, n, t_end, dt, seed, **kw):
    model = _model(spec)
    m = cwc_dyn.cwc_dyn_model_create(model)
    gpu = cwc_dyn.simulate(m, n, t_end, dt, seed, want_traj=True, **kw)
    torch.cuda.synchronize()
    traj, fir, st = oracle_runs(spec, t_end, dt, seed, list(range(n)))
    g_traj = gpu["traj"].cpu().numpy()
    g_st = gpu["status"].cpu().numpy()
    assert (g_st != cwc_dyn.CWC_TRAJ_CAPACITY).all(), "capacity reached in a parity case"
    same = (g_traj == traj).all(axis=(1, 2))
    assert same.all(), ("trajectory mismatch", spec, np.nonzero(~same)[0][:10])
    assert (gpu["firings"].cpu().numpy() == fir).all()
    assert (g_st == st).all()
    cnt, s1, s2 = _moments(traj)
    assert (gpu["count"].cpu().numpy() == cnt).all()
    assert (gpu["sum"].cpu().numpy() == s1.astype(np.int64)).all()
    sq = gpu["sumsq"].cpu().numpy().view(np.uint64)
    hi_lo = sq[..., 0].astype(object) + (sq[..., 1].astype(object) << 64)
    assert (hi_lo == s2).all()
    return gpu, traj


def test_cell_population_full_horizon():
    c = wd.CONFIG_C6
    _check(("cell", {}), 96, c["t_end"], c["sample_dt"], c["seed"])


@pytest.mark.parametrize("seed", RANDOM_SEEDS)
def test_random_models(seed):
    _check(("random", seed), 48, 6.0, 0.1, 3)


def test_launch_shape_invariance():
    model = wd.cell_population_model()
    m = cwc_dyn.cwc_dyn_model_create(model)
    ref = cwc_dyn.simulate(m, 200, 5.0, 0.1, 7, want_traj=True)
    ref_t = ref["traj"].cpu().clone()
    ref_sum = ref["sum"].cpu().clone()
    for wpb, bps in [(1, 1), (2, 3), (8, 0), (3, 2)]:
        r = cwc_dyn.simulate(m, 200, 5.0, 0.1, 7, want_traj=True, warps_per_block=wpb, blocks_per_sm=bps)
        assert torch.equal(r["traj"].cpu(), ref_t), (wpb, bps)
        assert torch.equal(r["sum"].cpu(), ref_sum)


def test_shard_equals_unsharded():
    model = wd.cell_population_model()
    m = cwc_dyn.cwc_dyn_model_create(model)
    full = cwc_dyn.simulate(m, 100, 4.0, 0.1, 5, want_traj=True)
    ft = full["traj"].cpu().clone()
    a = cwc_dyn.simulate(m, 40, 4.0, 0.1, 5, want_traj=True, replica_offset=0, replicas_total=100)
    at = a["traj"].cpu().clone()
    b = cwc_dyn.simulate(m, 60, 4.0, 0.1, 5, want_traj=True, replica_offset=40, replicas_total=100)
    assert torch.equal(at, ft[:40])
    assert torch.equal(b["traj"].cpu(), ft[40:])


def test_capacity_status():
    cap = 12
    m = cwc_dyn.cwc_dyn_model_create(creation_model())
    n, t_end, dt = 24, 10.0, 0.5
    gpu = cwc_dyn.simulate(m, n, t_end, dt, 1, want_traj=True, capacity=cap)
    torch.cuda.synchronize()
    traj, fir, st = oracle_runs(("creation", None), t_end, dt, 1, list(range(n)))
    g = gpu["traj"].cpu().numpy()
    gst = gpu["status"].cpu().numpy()
    hit = 0
    for i in range(n):
        over = np.nonzero(traj[i, :, 0] >= cap)[0]
        if len(over) == 0:   # this trajectory never needs more than the capacity: plain parity
            assert gst[i] == st[i] and (g[i] == traj[i]).all()
            continue
        hit += 1
        assert gst[i] == cwc_dyn.CWC_TRAJ_CAPACITY
        j0 = over[0]
        assert (g[i, :j0] == traj[i, :j0]).all()
        assert (g[i, j0:, 0] == cap - 1).all()          # frozen with capacity - 1 compartments
        assert (g[i, j0:] == g[i, j0]).all()
    assert hit >= n // 2


def test_stall_and_no_rules():
    # a term whose every rule stalls at once: samples = the initial term, status STALLED
    model = {"name": "stall", "n_atoms": 2, "n_labels": 2,
             "term": {"atoms": {0: 0}, "comps": [{"label": 1, "wrap": {1: 3}, "content": {"atoms": {0: 4}}}]},
             "rules": [{"label": 0, "atoms": {1: 1}, "rate": 1.0, "rhs": {"X": True, "atoms": {}}}],
             "observables": [("count", 1), ("wrap", 1, 1), ("content", 1, 0)]}
    m = cwc_dyn.cwc_dyn_model_create(model)
    r = cwc_dyn.simulate(m, 5, 1.0, 0.25, 1, want_traj=True)
    assert (r["status"].cpu().numpy() == 1).all()
    assert (r["firings"].cpu().numpy() == 0).all()
    assert (r["traj"].cpu().numpy() == np.array([1, 3, 4])).all()


def test_cell_population_survey_scale():
    """C6 at its bench launch shape (8192 replicas, full horizon) against the
    oracle on the trajectories g = 0 mod 16 (512); writes the parity report
    when CWC_PARITY_OUT names a directory."""
    import json
    c = wd.CONFIG_C6
    m = cwc_dyn.cwc_dyn_model_create(wd.cell_population_model())
    gpu = cwc_dyn.simulate(m, c["n_replicas"], c["t_end"], c["sample_dt"], c["seed"], want_traj=True)
    torch.cuda.synchronize()
    g_list = list(range(0, c["n_replicas"], 16))
    traj, fir, st = oracle_runs(("cell", {}), c["t_end"], c["sample_dt"], c["seed"], g_list)
    g_traj = gpu["traj"].cpu().numpy()[g_list]
    same = (g_traj == traj).all(axis=(1, 2))
    same &= gpu["firings"].cpu().numpy()[g_list] == fir
    same &= gpu["status"].cpu().numpy()[g_list] == st
    out = os.environ.get("CWC_PARITY_OUT")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "parity_C6.json"), "w") as f:
            json.dump({"config": "C6", "compared": len(g_list), "matched": int(same.sum()),
                       "firings_compared": int(fir.sum()), "divergent": [int(g_list[i]) for i in np.nonzero(~same)[0]]}, f)
    assert same.all(), ("divergent trajectories", [g_list[i] for i in np.nonzero(~same)[0]][:10])


def _overflow_models():
    big = 2**31 - 7
    # non-structural: influx at the top level pushes a count past int32
    influx = {"name": "overflow-influx", "n_atoms": 2, "n_labels": 2,
              "term": {"atoms": {0: big}, "comps": [{"label": 1, "wrap": {}, "content": {"atoms": {1: 3}}}]},
              "rules": [{"label": 0, "atoms": {}, "rate": 1.0, "rhs": {"X": True, "atoms": {0: 2}}},
                        {"label": 1, "atoms": {1: 1}, "rate": 0.5, "rhs": {"X": True, "atoms": {}}}],
              "observables": [("content", 0, 0), ("content", 1, 1), ("count", 1)]}
    # structural: lysis releases a cell's content into a top level that is near the limit
    lysis = {"name": "overflow-lysis", "n_atoms": 1, "n_labels": 2,
             "term": {"atoms": {0: big}, "comps": [{"label": 1, "wrap": {}, "content": {"atoms": {0: 5}}},
                                                   {"label": 1, "wrap": {}, "content": {"atoms": {0: 9}}}]},
             "rules": [{"label": 0, "atoms": {}, "rate": 0.7, "comp": {"label": 1, "wrap": {}, "content": {}},
                        "rhs": {"X": True, "atoms": {}, "release_W": True, "release_Y": True}},
                       {"label": 1, "atoms": {0: 1}, "rate": 0.3, "rhs": {"X": True, "atoms": {}}}],
             "observables": [("content", 0, 0), ("content", 1, 0), ("count", 1)]}
    return [influx, lysis]


@pytest.mark.parametrize("which", [0, 1], ids=["influx", "lysis"])
def test_overflow_status_matches_oracle(which):
    model = _overflow_models()[which]
    m = cwc_dyn.cwc_dyn_model_create(model)
    n, t_end, dt = 40, 8.0, 0.25
    gpu = cwc_dyn.simulate(m, n, t_end, dt, 2, want_traj=True)
    torch.cuda.synchronize()
    ora = dyn.simulate(model, 0, t_end, dt, 2, g_list=list(range(n)))
    assert (gpu["status"].cpu().numpy() == ora["status"]).all()
    assert (ora["status"] == 2).any()          # the case exercises OVERFLOW
    assert (gpu["traj"].cpu().numpy() == ora["traj"]).all()
    assert (gpu["firings"].cpu().numpy() == ora["firings"]).all()
