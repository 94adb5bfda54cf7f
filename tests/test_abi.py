"""CPU tests of the C-ABI library: it loads, exports every symbol cwc.h
declares, and its host logic (validation, flattening, dependency graph,
launch planning) is correct.  No kernel is launched here (no GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import workloads as w
from paper_1010_2438_b200 import cwc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1010_2438_b200 import _build
    _build.build()


def test_every_declared_symbol_is_exported():
    hdr = open(os.path.join(ROOT, "include", "cwc.h")).read()
    declared = set(re.findall(r"\b(cwc_[a-z0-9_]+)\s*\(", hdr))
    assert "cwc_simulate" in declared and "cwc_model_create" in declared
    L = cwc.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(cwc.EXPORTED) == declared


MODELS = [("paper", lambda: w.paper_example_model()), ("small_cwc", lambda: w.small_cwc_model(3, 1)),
          ("C1", lambda: w.config("C1")[0]), ("C2", lambda: w.config("C2")[0]), ("C3", lambda: w.config("C3")[0]),
          ("C4", lambda: w.config("C4")[0]), ("C5", lambda: w.config("C5")[0]),
          ("dimer", lambda: w.dimerisation_model())]


@pytest.mark.parametrize("name,make", MODELS)
def test_flattening_equals_oracle_flattening(name, make):
    d = make()
    m = cwc.cwc_model_create(d)
    f = m.get_flat()
    ent = oracle.flatten(d)
    assert m.info.n_reactions == len(ent)
    assert list(f["entry_rule"]) == [e["rule"] for e in ent]
    assert list(f["entry_context"]) == [e["context"] for e in ent]
    assert list(f["entry_child"]) == [e["child"] for e in ent]
    for k, e in enumerate(ent):
        lo, hi = f["re_ptr"][k], f["re_ptr"][k + 1]
        assert list(zip(f["re_cell"][lo:hi], f["re_mult"][lo:hi])) == [tuple(x) for x in e["reactants"]]
        lo, hi = f["nu_ptr"][k], f["nu_ptr"][k + 1]
        assert list(zip(f["nu_cell"][lo:hi], f["nu_delta"][lo:hi])) == [tuple(x) for x in e["nu"]]


@pytest.mark.parametrize("name,make", MODELS)
def test_dependency_graph_is_exact(name, make):
    d = make()
    m = cwc.cwc_model_create(d)
    f = m.get_flat()
    ent = oracle.flatten(d)
    reads = [set(c for c, _ in e["reactants"]) for e in ent]
    for mu, e in enumerate(ent):
        changed = set(c for c, _ in e["nu"])
        want = [k for k in range(len(ent)) if reads[k] & changed]
        got = list(f["dep"][f["dep_ptr"][mu]:f["dep_ptr"][mu + 1]])
        assert got == want, mu
    assert m.info.max_deps == max((f["dep_ptr"][i + 1] - f["dep_ptr"][i] for i in range(len(ent))), default=0)


def test_path_choice():
    assert cwc.cwc_model_create(w.config("C2")[0]).info.path == cwc.CWC_PATH_THREAD
    assert cwc.cwc_model_create(w.config("C3")[0]).info.path == cwc.CWC_PATH_THREAD
    assert cwc.cwc_model_create(w.config("C4")[0]).info.path == cwc.CWC_PATH_WARP
    assert cwc.cwc_model_create(w.config("C5")[0]).info.path == cwc.CWC_PATH_WARP


def _bad(mut):
    d = w.lotka_volterra_model()
    mut(d)
    with pytest.raises(cwc.CwcError) as ei:
        cwc.cwc_model_create(d)
    return ei.value.status


def test_model_validation_errors():
    R = w.models._rule
    assert _bad(lambda d: d["rules"][0].__setitem__("rate", 0.0)) == cwc.CWC_ERR_INVALID
    assert _bad(lambda d: d["rules"][0].__setitem__("rate", float("nan"))) == cwc.CWC_ERR_INVALID
    assert _bad(lambda d: d["rules"][0].__setitem__("rate", float("inf"))) == cwc.CWC_ERR_INVALID
    assert _bad(lambda d: d["init"].__setitem__(0, -1)) == cwc.CWC_ERR_INVALID
    assert _bad(lambda d: d["rules"].append(R(0, [(0, 0, 3)], [], 1.0))) == cwc.CWC_ERR_UNSUPPORTED
    assert _bad(lambda d: d["rules"].append(R(0, [(0, 0, 2), (0, 1, 1)], [], 1.0))) == cwc.CWC_ERR_UNSUPPORTED
    assert _bad(lambda d: d["rules"].append(R(0, [(1, 0, 1)], [], 1.0))) == cwc.CWC_ERR_INVALID  # child on local rule
    assert _bad(lambda d: d["rules"].append(R(0, [(0, 5, 1)], [], 1.0))) == cwc.CWC_ERR_INVALID  # species range
    assert _bad(lambda d: d["rules"].append(R(3, [], [], 1.0))) == cwc.CWC_ERR_INVALID  # label range
    assert _bad(lambda d: d["rules"].append(R(0, [(0, 0, 0)], [], 1.0))) == cwc.CWC_ERR_INVALID  # mult 0
    assert _bad(lambda d: d["obs_of_cell"].__setitem__(0, 7)) == cwc.CWC_ERR_INVALID


def test_tree_validation_errors():
    d = w.small_cwc_model(2)
    d["parent"][2] = 3  # parent index not < child index
    with pytest.raises(cwc.CwcError):
        cwc.cwc_model_create(d)
    d = w.small_cwc_model(2)
    d["type"][0] = 1
    with pytest.raises(cwc.CwcError):
        cwc.cwc_model_create(d)
    d = w.small_cwc_model(2)
    d["type"][1] = 9
    with pytest.raises(cwc.CwcError):
        cwc.cwc_model_create(d)


def test_run_argument_errors():
    m = cwc.cwc_model_create(w.config("C2")[0])
    for args in [(16, None, 0.0, 0.1), (16, None, -1.0, 0.1), (16, None, 1.0, 0.0), (16, None, 1.0, 2.0),
                 (0, None, 1.0, 0.1), (16, None, float("inf"), 0.1),
                 (16, {"rules": [7], "values": [[1.0]]}, 1.0, 0.1),
                 (16, {"rules": [0], "values": [[-1.0]]}, 1.0, 0.1),
                 (16, {"rules": [0], "values": []}, 1.0, 0.1)]:
        with pytest.raises(cwc.CwcError) as ei:
            cwc.cwc_simulate_workspace_size(m, *args)
        assert ei.value.status == cwc.CWC_ERR_INVALID, args
    opts = cwc.cwc_sim_opts()
    opts.force_path = cwc.CWC_PATH_THREAD
    big = cwc.cwc_model_create(w.config("C4")[0])
    with pytest.raises(cwc.CwcError):
        cwc.cwc_simulate_workspace_size(big, 16, None, 1.0, 0.1, opts)
    opts.force_path = cwc.CWC_PATH_AUTO
    opts.block_threads = 48
    with pytest.raises(cwc.CwcError):
        cwc.cwc_simulate_workspace_size(m, 16, None, 1.0, 0.1, opts)


def test_workspace_grows_with_work():
    m = cwc.cwc_model_create(w.config("C3")[0])
    d, sweep, cfg = w.config("C3")
    a = cwc.cwc_simulate_workspace_size(m, 16, sweep, 50.0, 0.5)
    b = cwc.cwc_simulate_workspace_size(m, 16, None, 50.0, 0.5)
    assert a > b > 0


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure mode")
def test_simulate_without_gpu_fails_loudly():
    import torch
    m = cwc.cwc_model_create(w.config("C1")[0])
    z = torch.zeros(8, dtype=torch.int64)
    ws = torch.zeros(1 << 20, dtype=torch.uint8)
    with pytest.raises(cwc.CwcError) as ei:
        cwc.cwc_simulate(m, 16, None, 10.0, 1.0, 1, 0, (z, z, z), ws)
    assert ei.value.status == cwc.CWC_ERR_CUDA
    with pytest.raises(RuntimeError):
        cwc.simulate(m, 16, 10.0, 1.0, 1)


def test_run_state_size_and_errors():
    """Resumable runs (cwc_run_*): the state buffer holds per-trajectory
    (x, t, n, j), two live lists and the accumulators; same argument checks
    as cwc_simulate; tracing is refused."""
    d, sweep, cfg = w.config("C3")
    m = cwc.cwc_model_create(d)
    G = 16 * len(sweep["values"])
    a = cwc.cwc_run_state_size(m, 16, sweep, 50.0, 0.5)
    assert a >= G * (4 * m.info.n_cells + 8 + 8 + 4 + 2 * 8)
    assert a > cwc.cwc_run_state_size(m, 16, None, 50.0, 0.5) > 0
    for args in [(16, None, 0.0, 0.1), (16, None, 1.0, 2.0), (0, None, 1.0, 0.1)]:
        with pytest.raises(cwc.CwcError) as ei:
            cwc.cwc_run_state_size(m, *args)
        assert ei.value.status == cwc.CWC_ERR_INVALID, args
    opts = cwc.cwc_sim_opts()
    g = np.zeros(1, dtype=np.int64)
    opts.trace_g = g.ctypes.data
    opts.n_trace = 1
    with pytest.raises(cwc.CwcError) as ei:
        cwc.cwc_run_state_size(m, 16, None, 1.0, 0.1, opts)
    assert ei.value.status == cwc.CWC_ERR_INVALID


def _opts(**kw):
    o = cwc.cwc_sim_opts()
    o.force_path = cwc.CWC_PATH_AUTO
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def test_plan_override_validation():
    """cwc_sim_opts plan overrides (kernel, stats_mode, warps_per_block,
    blocks_per_sm) are validated; nothing is read from the environment."""
    c2 = cwc.cwc_model_create(w.config("C2")[0])
    c5 = cwc.cwc_model_create(w.config("C5")[0])
    ok = [dict(kernel=cwc.CWC_KERNEL_THREAD_WS), dict(kernel=cwc.CWC_KERNEL_THREAD), dict(kernel=cwc.CWC_KERNEL_WARP2),
          dict(kernel=cwc.CWC_KERNEL_WARP), dict(stats_mode=cwc.CWC_STATS_GLOBAL), dict(stats_mode=cwc.CWC_STATS_SHARED),
          dict(kernel=cwc.CWC_KERNEL_WARP, warps_per_block=2, blocks_per_sm=3)]
    for kw in ok:
        assert cwc.cwc_simulate_workspace_size(c2, 64, None, 1.0, 0.1, _opts(**kw)) > 0, kw
    bad = [(c2, dict(kernel=9)), (c2, dict(kernel=-1)), (c2, dict(stats_mode=3)), (c2, dict(warps_per_block=5)),
           (c2, dict(warps_per_block=-1)), (c2, dict(blocks_per_sm=33)), (c2, dict(force_path=5)),
           (c2, dict(kernel=cwc.CWC_KERNEL_WARP, force_path=cwc.CWC_PATH_THREAD)),
           (c2, dict(kernel=cwc.CWC_KERNEL_THREAD_WS, force_path=cwc.CWC_PATH_WARP)),
           (c2, dict(kernel=cwc.CWC_KERNEL_THREAD_WS, block_threads=64)),
           (c5, dict(kernel=cwc.CWC_KERNEL_THREAD)),      # 264 cells: no thread path
           (c5, dict(kernel=cwc.CWC_KERNEL_WARP2)),       # M = 1172 > 256
           (c5, dict(kernel=cwc.CWC_KERNEL_WARP8)), (c5, dict(kernel=cwc.CWC_KERNEL_WARP4))]
    for m, kw in bad:
        with pytest.raises(cwc.CwcError) as ei:
            cwc.cwc_simulate_workspace_size(m, 64, None, 1.0, 0.1, _opts(**kw))
        assert ei.value.status == cwc.CWC_ERR_INVALID, kw
    # resumable runs: no warp-specialised kernel, no shared-memory parts
    for kw in (dict(kernel=cwc.CWC_KERNEL_THREAD_WS), dict(stats_mode=cwc.CWC_STATS_SHARED)):
        with pytest.raises(cwc.CwcError) as ei:
            cwc.cwc_run_state_size(c2, 64, None, 1.0, 0.1, _opts(**kw))
        assert ei.value.status == cwc.CWC_ERR_INVALID, kw


def test_environment_does_not_change_the_plan(monkeypatch):
    """The round-1 experiment variables are no longer read by release builds."""
    m = cwc.cwc_model_create(w.config("C4")[0])
    a = cwc.cwc_simulate_workspace_size(m, 64, None, 1.0, 0.1)
    for k, v in [("CWC_STATS_MODE", "smem"), ("CWC_WARP_SEG", "32"), ("CWC_WARPS_PER_BLOCK", "0"),
                 ("CWC_BLOCKS_PER_SM", "1"), ("CWC_FORCE_PATH", "0"), ("CWC_WS", "1"), ("CWC_PROF_PTR", "0x10")]:
        monkeypatch.setenv(k, v)
    assert cwc.cwc_simulate_workspace_size(m, 64, None, 1.0, 0.1) == a


def test_int64_moment_bound():
    """Per-cell observable sums over all replicas must fit int64:
    a run whose replicas could overflow them is refused."""
    m = cwc.cwc_model_create(w.config("C5")[0])   # observables < 2^36
    assert cwc.cwc_simulate_workspace_size(m, 8192, None, 1.0, 0.1) > 0
    with pytest.raises(cwc.CwcError) as ei:
        cwc.cwc_simulate_workspace_size(m, 16, None, 1.0, 0.1, _opts(replicas_total=2**28))
    assert ei.value.status == cwc.CWC_ERR_INVALID


def test_plan_reports_the_kernel_and_accumulators():
    """cwc_plan: the automatic plan per config (148 SMs assumed without a
    GPU): the warp-specialised thread kernel while at most two CTAs share an
    SM (C1), the single-warp thread kernel beyond (C2, C3), two trajectories
    per warp for M <= 256 (C4), one per warp above (C5); statistics layout
    consistent with the workspace size."""
    want = {"C1": cwc.CWC_KERNEL_THREAD_WS, "C2": cwc.CWC_KERNEL_THREAD, "C3": cwc.CWC_KERNEL_THREAD,
            "C4": cwc.CWC_KERNEL_WARP2, "C5": cwc.CWC_KERNEL_WARP}
    for name, k in want.items():
        d, sweep, cfg = w.config(name)
        m = cwc.cwc_model_create(d)
        p = cwc.cwc_plan(m, cfg["n_replicas"], sweep, cfg["t_end"], cfg["sample_dt"])
        assert p.kernel == k, name
        P = len(sweep["values"]) if sweep else 1
        assert p.n_stat_cells == P * (int(cfg["t_end"] / cfg["sample_dt"] + 1e-9) + 1) * m.info.n_obs
        assert p.workspace_bytes == cwc.cwc_simulate_workspace_size(m, cfg["n_replicas"], sweep, cfg["t_end"],
                                                                   cfg["sample_dt"])
        assert p.word_bytes in (4, 8) and p.words_per_cell >= 3 and p.n_parts >= 1
        assert p.part_cells >= p.n_stat_cells if not p.stats_shared else p.part_cells > 0
    m = cwc.cwc_model_create(w.config("C2")[0])
    assert cwc.cwc_plan(m, 64, None, 1.0, 0.1, _opts(kernel=cwc.CWC_KERNEL_WARP)).kernel == cwc.CWC_KERNEL_WARP
    assert cwc.cwc_plan(m, 64, None, 1.0, 0.1, _opts(force_path=cwc.CWC_PATH_WARP)).kernel == cwc.CWC_KERNEL_WARP8


def test_plan_picks_the_warp_kernel_by_network_size():
    """Planner (cwc_api.cpp): eight trajectories per warp up to 128 reactions,
    two per warp up to 256, one per warp beyond (tools/warp8_crossover.py);
    the 4-lane-group kernel never for resumable runs or shared-memory parts."""
    def kern(desc, **kw):
        o = cwc.cwc_sim_opts()
        o.force_path = cwc.CWC_PATH_WARP
        for k, v in kw.items():
            setattr(o, k, v)
        return cwc.cwc_plan(cwc.cwc_model_create(desc), 64, None, 1.0, 0.1, o).kernel
    assert kern(w.lotka_volterra_chain(16)) == cwc.CWC_KERNEL_WARP8
    assert kern(w.random_network_model(seed=1, n_species=64, n_reactions=128)) == cwc.CWC_KERNEL_WARP8
    assert kern(w.random_network_model(seed=1, n_species=64, n_reactions=129)) == cwc.CWC_KERNEL_WARP2
    assert kern(w.config("C4")[0]) == cwc.CWC_KERNEL_WARP2
    assert kern(w.config("C5")[0]) == cwc.CWC_KERNEL_WARP
    assert kern(w.lotka_volterra_chain(16), stats_mode=cwc.CWC_STATS_SHARED) == cwc.CWC_KERNEL_WARP2
    assert kern(w.config("C4")[0], kernel=cwc.CWC_KERNEL_WARP8) == cwc.CWC_KERNEL_WARP8
    with pytest.raises(cwc.CwcError):
        kern(w.config("C5")[0], kernel=cwc.CWC_KERNEL_WARP8)


def test_plan_of_a_model_without_rules_keeps_the_selection_rows():
    """A model with no rules (M = 0) still plans on every warp kernel, and the
    group kernels reserve one (zeroed) 16-row sub-chunk of propensities per
    warp: their selection reads rows [0, 16) of the chosen sub-chunk even for
    a trajectory that stalls at once (ssa_warp8.cu, NS >= 1)."""
    desc = w.decay_model(5, 1.0)
    desc["rules"] = []
    m = cwc.cwc_model_create(desc)
    assert m.info.n_reactions == 0
    for kern, lg in ((cwc.CWC_KERNEL_WARP8, 4), (cwc.CWC_KERNEL_WARP4, 8)):
        p = cwc.cwc_plan(m, 33, None, 2.0, 0.5, _opts(kernel=kern))
        assert p.kernel == kern
        warps = p.threads // 32
        rows = 8 * 16 * 32  # one sub-chunk of fp64 rows [16][32]
        per_warp = rows + 8 * 4 * 32 + 16 * 32 * (32 // lg) + 4 * (32 // lg) * (m.info.n_cells + 1)
        assert p.smem_bytes >= warps * per_warp, (kern, p.smem_bytes, warps, per_warp)
    for kern in (cwc.CWC_KERNEL_WARP, cwc.CWC_KERNEL_WARP2):
        assert cwc.cwc_plan(m, 33, None, 2.0, 0.5, _opts(kernel=kern)).kernel == kern
