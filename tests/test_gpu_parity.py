"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Bar (BASELINE north_star): species counts at every sample bit-exact for
>= 99.9% of trajectories under the same Philox streams, every divergence
traced (tests/tracer.py) to a last-ulp fp64 log or sum-order difference,
never to a BUG; merged moments over matched trajectories equal (exact
integers); mean/variance within 1e-9 relative.  Sizes: small cases the
oracle runs whole (several CTAs, ragged tails), and BASELINE's full configs
in the bench launch shape with oracle-sampled trajectories.
"""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import workloads as w  # noqa: E402

from .tracer import trace_mismatches  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1010_2438_b200 import cwc  # noqa: E402

MIN_MATCH = 0.999


def _gpu(model, cfg, sweep=None, **kw):
    out = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep, **kw)
    torch.cuda.synchronize()
    return out


def _assert_moments_equal_dump(gpu, P, R):
    """The kernel's on-line moments equal an independent reduction of its own
    trajectory dump (int64 torch sums on the device: exact, bounds checked)."""
    t = gpu["traj"].view(P, R, gpu["traj"].shape[1], gpu["traj"].shape[2])
    vmax = int(t.abs().max().item()) if t.numel() else 0
    assert vmax * vmax * R < 2**62, "dump too large for exact int64 check"
    assert (gpu["count"] == R).all()
    assert torch.equal(gpu["sum"], t.sum(dim=1))
    assert (gpu["sumsq"][..., 1] == 0).all()
    assert torch.equal(gpu["sumsq"][..., 0], (t * t).sum(dim=1))


def _check_parity(desc, model, cfg, sweep, gpu, g_list, force_path, warp_path, **kw):
    """Compare trajectories with the oracle; trace every mismatch with the
    same kernel variant (kw: the run's plan overrides)."""
    ora = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                          g_list=g_list, want_stats=False)
    gt = gpu["traj"][torch.as_tensor(np.asarray(g_list), device="cuda")].cpu().numpy()
    gf = gpu["firings"][torch.as_tensor(np.asarray(g_list), device="cuda")].cpu().numpy()
    gs = gpu["status"][torch.as_tensor(np.asarray(g_list), device="cuda")].cpu().numpy()
    same = np.array([(gt[i] == ora["traj"][i]).all() for i in range(len(g_list))])
    same &= (gf == ora["firings"]) | ~same
    bad_i = list(np.nonzero(~same)[0])
    report = trace_mismatches(model, desc, sweep, cfg, [g_list[i] for i in bad_i], warp_path, force_path,
                              gpu_rows=[gt[i] for i in bad_i], ora_rows=[ora["traj"][i] for i in bad_i],
                              **kw) if bad_i else []
    for rec in report:
        assert rec[1] not in ("BUG", "identical-trace"), rec
    assert same.mean() >= MIN_MATCH, (same.mean(), report)
    matched = np.nonzero(same)[0]
    assert (gf[matched] == ora["firings"][matched]).all()
    assert (gs[matched] == ora["status"][matched]).all()
    return same, report, ora


# ---------------------------------------------------------------------------
# RNG
# ---------------------------------------------------------------------------

def test_device_philox_matches_oracle():
    rng = np.random.default_rng(0)
    g = rng.integers(0, 2**62, size=4096, dtype=np.int64)
    n = rng.integers(0, 2**62, size=4096, dtype=np.int64)
    g[:4] = [0, 1, 2**62 - 1, 16383]
    n[:4] = [0, 0, 5, 300000]
    out = torch.zeros((4096, 4), dtype=torch.int32, device="cuda")
    for seed in (1, 0xFFFFFFFFFFFF1234):
        cwc.cwc_philox_blocks(seed, torch.as_tensor(g, device="cuda"), torch.as_tensor(n, device="cuda"), out,
                              torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        for i in range(0, 4096, 37):
            gi, ni = int(g[i]), int(n[i])
            want = oracle.philox4x32_10([ni & 0xFFFFFFFF, ni >> 32, gi & 0xFFFFFFFF, gi >> 32],
                                        [seed & 0xFFFFFFFF, seed >> 32])
            assert list(got[i]) == want


# ---------------------------------------------------------------------------
# thread path, small sizes: whole oracle, several CTAs + ragged tail
# ---------------------------------------------------------------------------

SMALL = [
    ("C1", lambda: (w.config("C1")[0], None), dict(t_end=100.0, sample_dt=1.0, n_replicas=1000, seed=1)),
    ("C2", lambda: (w.config("C2")[0], None), dict(t_end=2.0, sample_dt=0.01, n_replicas=300, seed=1)),
    ("C3", lambda: (w.config("C3")[0], w.mm_sweep(5, 7)), dict(t_end=50.0, sample_dt=0.5, n_replicas=13, seed=1)),
    ("decay", lambda: (w.decay_model(1000, 1.0), None), dict(t_end=1.0, sample_dt=0.25, n_replicas=777, seed=3)),
    ("stall", lambda: (w.decay_model(3, 5.0), None), dict(t_end=10.0, sample_dt=1.0, n_replicas=65, seed=4)),
    ("dimer", lambda: (w.dimerisation_model(50, 0.1), None), dict(t_end=3.0, sample_dt=0.1, n_replicas=129, seed=8)),
    ("paper", lambda: (w.paper_example_model(0.5), None), dict(t_end=5.0, sample_dt=0.5, n_replicas=40, seed=2)),
    ("one", lambda: (w.config("C1")[0], None), dict(t_end=3.0, sample_dt=3.0, n_replicas=1, seed=5)),
    # thread-path batch widths 2 and 1 (M in 9..16 and 17..32), all 8 register cells
    ("rnd12", lambda: (w.random_network_model(seed=3, n_species=6, n_reactions=12), None),
     dict(t_end=0.5, sample_dt=0.05, n_replicas=70, seed=2)),
    ("rnd24", lambda: (w.random_network_model(seed=5, n_species=8, n_reactions=24), None),
     dict(t_end=0.2, sample_dt=0.02, n_replicas=45, seed=3)),
    # n-species Lotka-Volterra family (NEXT-2): 4 species (both paths), 16 (warp path)
    ("lv4", lambda: (w.lotka_volterra_chain(4), None), dict(t_end=0.3, sample_dt=0.01, n_replicas=70, seed=6)),
    ("lv16", lambda: (w.lotka_volterra_chain(16), None), dict(t_end=0.1, sample_dt=0.01, n_replicas=40, seed=7)),
    # warp path with B > 16 reactions per lane (one-trajectory kernel): M = 525
    ("cwc130", lambda: (w.small_cwc_model(130, 2), None), dict(t_end=0.5, sample_dt=0.05, n_replicas=40, seed=4)),
    # one-trajectory warp kernel with 33 reactions per lane (paired one-pass selection): M = 1045
    ("cwc260", lambda: (w.small_cwc_model(260, 3), None), dict(t_end=0.4, sample_dt=0.05, n_replicas=40, seed=5)),
]


KERNELS = [("thread", cwc.CWC_PATH_THREAD, {"kernel": cwc.CWC_KERNEL_THREAD_WS}),  # warp-specialised thread kernel
           ("thread1", cwc.CWC_PATH_THREAD, {"block_threads": 64, "kernel": cwc.CWC_KERNEL_THREAD}),  # single-warp, 1/lane
           ("thread2", cwc.CWC_PATH_THREAD, {"kernel": cwc.CWC_KERNEL_THREAD2}),  # single-warp, 2 trajectories per lane
           ("ws2", cwc.CWC_PATH_THREAD, {"kernel": cwc.CWC_KERNEL_THREAD_WS2}),   # warp-specialised, 2 per lane
           ("warp", cwc.CWC_PATH_WARP, {}),                           # the planner's warp kernel
           ("warp2", cwc.CWC_PATH_WARP, {"kernel": cwc.CWC_KERNEL_WARP2}),  # two trajectories per warp (M <= 256)
           ("warp32", cwc.CWC_PATH_WARP, {"kernel": cwc.CWC_KERNEL_WARP}),  # one trajectory per warp
           ("warp8", cwc.CWC_PATH_WARP, {"kernel": cwc.CWC_KERNEL_WARP8}),  # eight per warp (M <= 256)
           ("warp4", cwc.CWC_PATH_WARP, {"kernel": cwc.CWC_KERNEL_WARP4})]  # four per warp (M <= 256)


@pytest.mark.parametrize("name,make,cfg", SMALL, ids=[s[0] for s in SMALL])
@pytest.mark.parametrize("kname,path,kw", KERNELS, ids=[k[0] for k in KERNELS])
def test_small_parity_full_oracle(name, make, cfg, kname, path, kw):
    kw = dict(kw)
    if name in ("cwc130", "cwc260", "lv16") and path == cwc.CWC_PATH_THREAD:
        pytest.skip("more than 8 cells: warp path only")
    if name in ("rnd12", "rnd24") and kname in ("thread2", "ws2"):
        pytest.skip("two trajectories per lane: M <= 8 only")
    if name in ("cwc130", "cwc260") and kname in ("warp8", "warp4", "warp2"):
        pytest.skip("4-lane groups / 16-lane segments: M <= 256 only")
    desc, sweep = make()
    model = cwc.cwc_model_create(desc)
    gpu = _gpu(model, cfg, sweep, want_traj=True, force_path=path, **kw)
    P = gpu["n_points"]
    G = P * cfg["n_replicas"]
    same, report, ora = _check_parity(desc, model, cfg, sweep, gpu, list(range(G)), path, path == cwc.CWC_PATH_WARP,
                                      **kw)
    # moments: GPU on-line stats == reduction of the GPU's own dump (exact)
    _assert_moments_equal_dump(gpu, P, cfg["n_replicas"])
    if same.all():  # and == oracle's own on-line moments
        o = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                            want_traj=False)
        assert (gpu["count"].cpu().numpy() == o["count"]).all()
        assert (gpu["sum"].cpu().numpy() == o["sum"]).all()
        assert (gpu["sumsq"].cpu().numpy().view(np.uint64) == o["sumsq"]).all()


def test_overflow_status():
    desc = w.immigration_death_model(k_in=1e6, k_out=1e-12, a0=2**31 - 5)
    cfg = dict(t_end=1.0, sample_dt=0.5, n_replicas=40, seed=1)
    for path in (cwc.CWC_PATH_THREAD, cwc.CWC_PATH_WARP):
        gpu = _gpu(cwc.cwc_model_create(desc), cfg, want_traj=True, force_path=path)
        assert (gpu["status"].cpu().numpy() == cwc.CWC_TRAJ_OVERFLOW).all()
        assert (gpu["firings"].cpu().numpy() == 4).all()
        assert (gpu["traj"][:, -1, 0].cpu().numpy() == 2**31 - 1).all()


def test_no_rules_stalls_immediately():
    desc = w.decay_model(5, 1.0)
    desc["rules"] = []
    cfg = dict(t_end=2.0, sample_dt=0.5, n_replicas=33, seed=1)
    for path in (cwc.CWC_PATH_THREAD, cwc.CWC_PATH_WARP):
        gpu = _gpu(cwc.cwc_model_create(desc), cfg, want_traj=True, force_path=path)
        assert (gpu["status"].cpu().numpy() == cwc.CWC_TRAJ_STALLED).all()
        assert (gpu["traj"].cpu().numpy() == 5).all()
        assert (gpu["count"].cpu().numpy() == 33).all()


@pytest.mark.parametrize("bt", [32, 64, 96, 160, 256])
def test_launch_shape_does_not_change_results(bt):
    desc, _, _ = w.config("C2")
    cfg = dict(t_end=1.0, sample_dt=0.01, n_replicas=1111, seed=7)
    model = cwc.cwc_model_create(desc)
    ref = _gpu(model, cfg, block_threads=0)
    got = _gpu(model, cfg, block_threads=bt)
    for k in ("count", "sum", "sumsq", "firings", "status"):
        assert torch.equal(ref[k], got[k]), k


@pytest.mark.parametrize("mode", [cwc.CWC_STATS_SHARED, cwc.CWC_STATS_GLOBAL])
def test_stats_modes_agree(mode):
    desc, sweep, _ = w.config("C3")
    sweep = w.mm_sweep(6, 6)
    cfg = dict(t_end=20.0, sample_dt=0.5, n_replicas=40, seed=1)
    model = cwc.cwc_model_create(desc)
    ref = _gpu(model, cfg, sweep)
    for path in (cwc.CWC_PATH_THREAD, cwc.CWC_PATH_WARP):
        got = _gpu(model, cfg, sweep, force_path=path, stats_mode=mode)
        for k in ("count", "sum", "sumsq"):
            assert torch.equal(ref[k], got[k]), (mode, path, k)


def test_finalize_matches_oracle_moments():
    """Mean, variance and ci90 of a run equal the oracle's bit for bit: the
    device forms every quotient exactly and rounds it once (cwc.h,
    cwc_stats_finalize), like the oracle's Fraction -> float."""
    desc, _, _ = w.config("C1")
    cfg = dict(t_end=100.0, sample_dt=1.0, n_replicas=1024, seed=1)
    gpu = _gpu(cwc.cwc_model_create(desc), cfg, finalize=True)
    o = oracle.simulate(desc, 1024, 100.0, 1.0, 1, want_traj=False)
    means, vars_, cis = oracle.finalize(o["count"], o["sum"], o["sumsq"])
    for got, want in ((gpu["mean"], means), (gpu["var"], vars_), (gpu["ci90"], cis)):
        g = got.cpu().numpy().reshape(-1)
        wv = np.asarray(want, dtype=np.float64)
        assert np.array_equal(g.view(np.uint64), wv.view(np.uint64))


def test_finalize_exact_rounding_on_wide_moments():
    """cwc_stats_finalize on synthetic moment cells spanning the whole
    accumulator range (counts to 2^40, sums to 2^63, 128-bit sums of
    squares; numerators and denominators far beyond 2^53, tiny and huge
    quotients, exact and halfway cases): mean and variance equal the
    oracle's correctly rounded Fraction quotients bit for bit."""
    rng = np.random.default_rng(7)
    cells = []  # (n, s1, s2) Python ints with n*s2 >= s1^2
    # values v_i in a block: n copies split between a and b  ->  exact moments
    for _ in range(300):
        n = int(rng.integers(2, 1 << int(rng.integers(2, 41))))
        a = int(rng.integers(0, 1 << int(rng.integers(1, 24))))
        b = a + int(rng.integers(0, 1 << int(rng.integers(1, 23))))
        k = int(rng.integers(0, n + 1))  # k values equal a, n - k equal b
        s1 = k * a + (n - k) * b
        s2 = k * a * a + (n - k) * b * b
        if s1 < (1 << 63):
            cells.append((n, s1, s2))
    # hand-made: zero variance, count 1, count 0, halfway quotients, huge s2
    cells += [(5, 35, 245), (1, 7, 49), (0, 0, 0), (2, 1, 1), (3, 1, 1), (2, (1 << 53) + 1, ((1 << 53) + 1) ** 2),
              (1 << 40, (1 << 62) + 12345, ((1 << 84) + 999) + (1 << 100)), (3, 2**53 + 1, (2**53 + 1) ** 2),
              (7, 6, 36), (1 << 20, 3, 9), ((1 << 40) - 1, (1 << 40) - 1, (1 << 40) - 1)]
    cells = [c for c in cells if c[0] * c[2] >= c[1] * c[1]]
    n = len(cells)
    cnt = torch.tensor([c[0] for c in cells], dtype=torch.int64, device="cuda")
    s1 = torch.tensor([c[1] for c in cells], dtype=torch.int64, device="cuda")
    lo = np.array([c[2] & ((1 << 64) - 1) for c in cells], dtype=np.uint64)
    hi = np.array([c[2] >> 64 for c in cells], dtype=np.uint64)
    sq = torch.from_numpy(np.stack([lo, hi], axis=1).view(np.int64).copy()).cuda()
    mean = torch.empty(n, dtype=torch.float64, device="cuda")
    var = torch.empty_like(mean)
    ci = torch.empty_like(mean)
    cwc.cwc_stats_finalize((cnt, s1, sq), n, mean, var, ci, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    gm, gv, gc = mean.cpu().numpy(), var.cpu().numpy(), ci.cpu().numpy()
    for i, (c, a, b) in enumerate(cells):
        m, v, z = oracle.moments.finalize_cell(c, a, b)
        for got, want in ((gm[i], m), (gv[i], v), (gc[i], z)):
            if math.isnan(want):
                assert math.isnan(got), (cells[i], got)
            else:
                assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (cells[i], got, want)


@pytest.mark.parametrize("kern", [cwc.CWC_KERNEL_WARP2, cwc.CWC_KERNEL_WARP, cwc.CWC_KERNEL_WARP8,
                                  cwc.CWC_KERNEL_WARP4])
def test_trace_warp_paths_against_oracle(kern):
    """The warp kernels' per-firing traces (n, a0, tau, t', mu) against the
    oracle's: identical or differing only by the classified ulp-level
    reasons (sum order of a0 / the chunk prefixes, log ulp), never BUG."""
    desc = w.random_network_model(seed=5, n_species=8, n_reactions=24)
    cfg = dict(t_end=0.2, sample_dt=0.02, n_replicas=20, seed=3)
    model = cwc.cwc_model_create(desc)
    rep = trace_mismatches(model, desc, None, cfg, [0, 7, 19], True, cwc.CWC_PATH_WARP, kernel=kern)
    for g, cat, idx, detail in rep:
        assert cat in ("identical-trace", "log-ulp", "a0-sum-order", "select-order"), (g, cat, idx, detail)


def test_trace_equals_oracle_trace_thread_path():
    desc, _, _ = w.config("C2")
    cfg = dict(t_end=0.5, sample_dt=0.01, n_replicas=64, seed=1)
    model = cwc.cwc_model_create(desc)
    rep = trace_mismatches(model, desc, None, cfg, [0, 17, 63], False, cwc.CWC_PATH_THREAD)
    for g, cat, idx, detail in rep:
        assert cat in ("identical-trace", "log-ulp"), (g, cat, idx, detail)


@pytest.mark.parametrize("kern", [cwc.CWC_KERNEL_THREAD_WS, cwc.CWC_KERNEL_THREAD, cwc.CWC_KERNEL_THREAD2,
                                  cwc.CWC_KERNEL_THREAD_WS2])
def test_traced_thread_kernels_equal_untraced_and_each_other(kern):
    """Trace writes compiled into a thread kernel change nothing it computes,
    and both thread kernels (warp-specialised and single-warp, fast batches
    included) write the same per-firing records."""
    desc, _, _ = w.config("C2")
    cfg = dict(t_end=0.3, sample_dt=0.01, n_replicas=96, seed=4)
    model = cwc.cwc_model_create(desc)
    args = (model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"])
    plain = _gpu(model, cfg, kernel=kern)
    tr = cwc.simulate(*args, trace_g=[0, 33, 95], trace_cap=20000, kernel=kern)
    ref = cwc.simulate(*args, trace_g=[0, 33, 95], trace_cap=20000, kernel=cwc.CWC_KERNEL_THREAD_WS)
    torch.cuda.synchronize()
    for k in ("count", "sum", "sumsq", "firings", "status"):
        assert torch.equal(plain[k], tr[k]), k
    assert torch.equal(tr["trace_len"], ref["trace_len"])
    assert (tr["trace_len"].cpu() == tr["firings"][[0, 33, 95]].cpu() + 1).all()  # + the final drawn block
    assert torch.equal(tr["trace"], ref["trace"])


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_sharded_run_equals_unsharded(name):
    """replicas split over calls (as over GPUs: replica_offset /
    replicas_total) reproduce the unsharded trajectories; the exact integer
    moments of the shards sum to the unsharded moments bit for bit."""
    desc, sweep, _ = w.config(name)
    cfg = dict(t_end=0.3 if name == "C2" else 0.05, sample_dt=0.01, n_replicas=96, seed=5)
    model = cwc.cwc_model_create(desc)
    full = _gpu(model, cfg, sweep)
    parts = []
    for off, R in ((0, 40), (40, 56)):
        c = dict(cfg, n_replicas=R)
        parts.append(_gpu(model, c, sweep, replica_offset=off, replicas_total=96))
    assert torch.equal(torch.cat([p["firings"] for p in parts]), full["firings"])
    assert torch.equal(parts[0]["count"] + parts[1]["count"], full["count"])
    assert torch.equal(parts[0]["sum"] + parts[1]["sum"], full["sum"])
    lo = parts[0]["sumsq"][..., 0].view(torch.int64) + parts[1]["sumsq"][..., 0].view(torch.int64)
    assert torch.equal(lo, full["sumsq"][..., 0].view(torch.int64))  # no carry at these sizes


def test_host_output_api_equals_device_output():
    """cwc_simulate_host (host buffers, H2D/D2H inside the call) returns the
    same statistics as cwc_simulate with device buffers."""
    desc, sweep, _ = w.config("C3")
    sweep = w.mm_sweep(4, 4)
    cfg = dict(t_end=10.0, sample_dt=0.5, n_replicas=24, seed=3)
    model = cwc.cwc_model_create(desc)
    dev = _gpu(model, cfg, sweep)
    P, J1, O = dev["count"].shape
    hc = torch.empty(P * J1 * O, dtype=torch.int64, pin_memory=True)
    hs = torch.empty_like(hc)
    hq = torch.empty((P * J1 * O, 2), dtype=torch.int64, pin_memory=True)
    ws = torch.empty(cwc.cwc_simulate_host_workspace_size(model, cfg["n_replicas"], sweep, cfg["t_end"],
                                                         cfg["sample_dt"]), dtype=torch.uint8, device="cuda")
    cwc.cwc_simulate_host(model, cfg["n_replicas"], sweep, cfg["t_end"], cfg["sample_dt"], cfg["seed"],
                          torch.cuda.current_stream().cuda_stream, (hc, hs, hq), ws)
    torch.cuda.synchronize()
    assert torch.equal(hc.view(P, J1, O), dev["count"].cpu())
    assert torch.equal(hs.view(P, J1, O), dev["sum"].cpu())
    assert torch.equal(hq.view(P, J1, O, 2), dev["sumsq"].cpu())


@pytest.mark.parametrize("name,R,t_end", [("C2", 40000, 0.05), ("C3", 700, 5.0)])
def test_thread_kernels_agree_bitwise_multiwave(name, R, t_end):
    """The warp-specialised and the single-warp thread kernels compute the same
    trajectories bit for bit, also when the grid needs several waves of CTAs
    (C2: 40000 replicas; C3: 4096 points x 700 replicas, longest-first
    dispatch): identical moments, firings and statuses."""
    desc, sweep, _ = w.config(name)
    cfg = dict(t_end=t_end, sample_dt=t_end / 5, n_replicas=R, seed=9)
    model = cwc.cwc_model_create(desc)
    a = _gpu(model, cfg, sweep, kernel=cwc.CWC_KERNEL_THREAD_WS)
    b = _gpu(model, cfg, sweep, kernel=cwc.CWC_KERNEL_THREAD)
    c = _gpu(model, cfg, sweep, kernel=cwc.CWC_KERNEL_THREAD2)
    d = _gpu(model, cfg, sweep, kernel=cwc.CWC_KERNEL_THREAD_WS2)
    for k in ("count", "sum", "sumsq", "firings", "status"):
        assert torch.equal(a[k], b[k]), k
        assert torch.equal(a[k], c[k]), k
        assert torch.equal(a[k], d[k]), k
