"""GPU: resumable runs (cwc_run_*, the paper's time-sliced
schemas (ii)/(iii)).

A trajectory's progress is (x, t, n, j) and the RNG is keyed by (g, n), so a
run split into any sequence of advances -- firing quanta, sample windows,
both, with a checkpoint copied through host memory -- must reproduce the
one-shot run exactly: moments, firings, status and every sampled value.
The one-shot kernels are pinned to the oracle in test_gpu_parity.py; one
case here is also compared with the oracle directly.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import workloads as w  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1010_2438_b200 import cwc  # noqa: E402

CASES = [
    ("C2", lambda: (w.config("C2")[0], None), dict(t_end=1.0, sample_dt=0.01, n_replicas=300, seed=1)),
    ("C3", lambda: (w.config("C3")[0], w.mm_sweep(5, 7)), dict(t_end=50.0, sample_dt=0.5, n_replicas=13, seed=1)),
    ("stall", lambda: (w.decay_model(3, 5.0), None), dict(t_end=10.0, sample_dt=1.0, n_replicas=65, seed=4)),
    ("dimer", lambda: (w.dimerisation_model(50, 0.1), None), dict(t_end=3.0, sample_dt=0.1, n_replicas=129, seed=8)),
    ("rnd24", lambda: (w.random_network_model(seed=5, n_species=8, n_reactions=24), None),
     dict(t_end=0.2, sample_dt=0.02, n_replicas=45, seed=3)),
    ("cwc130", lambda: (w.small_cwc_model(130, 2), None), dict(t_end=0.3, sample_dt=0.05, n_replicas=40, seed=4)),
]

KERNELS = [("thread", cwc.CWC_PATH_THREAD, cwc.CWC_KERNEL_AUTO),
           ("warp", cwc.CWC_PATH_WARP, cwc.CWC_KERNEL_AUTO),   # two trajectories per warp (M <= 256)
           ("warp32", cwc.CWC_PATH_WARP, cwc.CWC_KERNEL_WARP)]  # one trajectory per warp


def _schedules(J1):
    wins = [max(1, J1 // 3), max(1, (2 * J1) // 3), J1]
    return [("q7", dict(quantum=7)), ("q200", dict(quantum=200)), ("windows", dict(windows=wins)),
            ("windows_q50", dict(quantum=50, windows=wins))]


def _equal(a, b, keys=("count", "sum", "sumsq", "firings", "status", "traj")):
    for k in keys:
        assert torch.equal(a[k], b[k]), k


@pytest.mark.parametrize("name,make,cfg", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("kname,path,kern", KERNELS, ids=[k[0] for k in KERNELS])
def test_resumable_equals_one_shot(name, make, cfg, kname, path, kern):
    desc, sweep = make()
    model = cwc.cwc_model_create(desc)
    if path == cwc.CWC_PATH_THREAD and not model.info.thread_path_ok:
        pytest.skip("more than 8 cells: warp path only")
    args = (model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
    one = cwc.simulate(*args, sweep=sweep, want_traj=True, force_path=path, kernel=kern)
    torch.cuda.synchronize()
    J1 = one["J1"]
    for sname, sch in _schedules(J1):
        res = cwc.simulate_resumable(*args, sweep=sweep, want_traj=True, force_path=path, kernel=kern, **sch)
        torch.cuda.synchronize()
        _equal(one, res)
        assert res["live"][-1] == 0
        if sname == "q7" and int(one["firings"].max()) > 3 * 32:
            assert res["advances"] > 2, res["live"]


def test_resumable_matches_oracle_directly():
    desc, cfg = w.config("C2")[0], dict(t_end=0.5, sample_dt=0.01, n_replicas=64, seed=3)
    model = cwc.cwc_model_create(desc)
    res = cwc.simulate_resumable(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], quantum=25,
                                 windows=[10, 30, 51], want_traj=True)
    torch.cuda.synchronize()
    ora = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
    same = (res["traj"].cpu().numpy() == ora["traj"]).all(axis=(1, 2))
    assert same.mean() >= 0.999
    if same.all():
        assert (res["firings"].cpu().numpy() == ora["firings"]).all()
        assert (res["count"].cpu().numpy() == ora["count"]).all()
        assert (res["sum"].cpu().numpy() == ora["sum"]).all()
        assert (res["sumsq"].cpu().numpy().view(np.uint64) == ora["sumsq"]).all()


@pytest.mark.parametrize("path", [cwc.CWC_PATH_THREAD, cwc.CWC_PATH_WARP])
def test_checkpoint_through_host_memory(path):
    """The state buffer is the whole run: copy it to host after an advance,
    drop the device copy, restore it into a fresh allocation and continue."""
    desc, sweep, _ = w.config("C3")
    sweep = w.mm_sweep(3, 4)
    cfg = dict(t_end=20.0, sample_dt=0.5, n_replicas=20, seed=11)
    model = cwc.cwc_model_create(desc)
    args = (model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
    one = cwc.simulate(*args, sweep=sweep, want_traj=True, force_path=path)
    torch.cuda.synchronize()
    saved = {}

    def ckpt(state, k):
        if k == 2:
            host = state.cpu()
            saved["bytes"] = host.numel()
            state.fill_(0xA5)  # the old buffer is garbage from here on
            return host.to("cuda")
        return None

    res = cwc.simulate_resumable(*args, sweep=sweep, quantum=300, want_traj=True, force_path=path, checkpoint=ckpt)
    torch.cuda.synchronize()
    assert saved["bytes"] > 0 and res["advances"] > 2
    _equal(one, res)


@pytest.mark.parametrize("path", [cwc.CWC_PATH_THREAD, cwc.CWC_PATH_WARP])
def test_windows_are_final_when_reached(path):
    """Schema (iii): after the advance to sample bound js, every trajectory
    sits at js (pending count 0), statuses read RUNNING, and the statistics of
    samples < js are already the final ones."""
    desc = w.config("C2")[0]
    cfg = dict(t_end=1.0, sample_dt=0.01, n_replicas=200, seed=5)
    model = cwc.cwc_model_create(desc)
    args = (model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
    one = cwc.simulate(*args, force_path=path)
    torch.cuda.synchronize()
    wins = [1, 17, 50, 99, 101]
    seen = []
    opts = cwc.cwc_sim_opts()
    opts.force_path = path

    def ckpt(state, k):
        js = wins[k - 1]
        n_cells = one["count"].numel() // 1
        c = torch.empty(n_cells, dtype=torch.int64, device="cuda")
        s = torch.empty_like(c)
        q = torch.empty((n_cells, 2), dtype=torch.int64, device="cuda")
        cwc.cwc_run_stats(model, cfg["n_replicas"], None, cfg["t_end"], cfg["sample_dt"], state, (c, s, q),
                          torch.cuda.current_stream().cuda_stream, opts)
        torch.cuda.synchronize()
        O = one["count"].shape[2]
        c, s, q = c.view(1, -1, O), s.view(1, -1, O), q.view(1, -1, O, 2)
        assert torch.equal(c[:, :js], one["count"][:, :js])
        assert torch.equal(s[:, :js], one["sum"][:, :js])
        assert torch.equal(q[:, :js], one["sumsq"][:, :js])
        if js < 101:
            assert (c[:, js:] == 0).all()  # nothing recorded past the bound
        seen.append(js)

    res = cwc.simulate_resumable(*args, windows=wins, force_path=path, checkpoint=ckpt)
    torch.cuda.synchronize()
    assert seen == wins and res["live"] == [0] * len(wins)
    _equal(one, res, keys=("count", "sum", "sumsq", "firings", "status"))


def test_overflow_and_stall_survive_suspension():
    cfg = dict(t_end=1.0, sample_dt=0.25, n_replicas=40, seed=1)
    for desc in (w.immigration_death_model(k_in=1e6, k_out=1e-12, a0=2**31 - 5), w.decay_model(3, 5.0)):
        model = cwc.cwc_model_create(desc)
        for path in (cwc.CWC_PATH_THREAD, cwc.CWC_PATH_WARP):
            args = (model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
            one = cwc.simulate(*args, want_traj=True, force_path=path)
            res = cwc.simulate_resumable(*args, quantum=1, windows=[2, 3, 5], want_traj=True, force_path=path)
            torch.cuda.synchronize()
            _equal(one, res)


@pytest.mark.parametrize("path", [cwc.CWC_PATH_THREAD, cwc.CWC_PATH_WARP])
def test_resumable_shard_equals_one_shot_shard(path):
    """A resumable run of one replica shard (replica_offset / replicas_total,
    SURVEY 8(e)) reproduces the one-shot run of the same shard."""
    desc, sweep = w.config("C3")[0], w.mm_sweep(3, 3)
    cfg = dict(t_end=20.0, sample_dt=0.5, n_replicas=7, seed=2)
    model = cwc.cwc_model_create(desc)
    args = (model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
    kw = dict(sweep=sweep, want_traj=True, force_path=path, replica_offset=5, replicas_total=16)
    one = cwc.simulate(*args, **kw)
    res = cwc.simulate_resumable(*args, quantum=100, windows=[11, 41], **kw)
    torch.cuda.synchronize()
    _equal(one, res)
