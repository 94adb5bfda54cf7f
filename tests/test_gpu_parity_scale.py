"""GPU parity at the survey's scale: BASELINE's five full configs in the bench
launch shape (the automatic plan -- the kernels bench.py times) against the
CPU oracle on deterministic trajectory subsets:

    C1  all 1024 trajectories          C4  g = 0 mod 32  (1024 of 32768)
    C2  g = 0 mod 8   (2048 of 16384)  C5  g = 0 mod 32  (256 of 8192)
    C3  g = 0 mod 16  (4096 of 65536)

Bar (BASELINE north_star): counts at every sample, firings and status
bit-exact for >= 99.9 % of the compared trajectories; every divergence
traced with the same kernel variant and classified with a VERIFIED
ulp-level cause (tests/tracer.py), never BUG; mean and variance over the
matched trajectories within 1e-9 relative of the oracle's.  Also: the
kernel's on-line moments equal the exact reduction of its own dump for every
trajectory, and the dump run's moments equal the bench call's.

The oracle runs in a process pool over the host's cores (spawned processes:
they import only oracle/ and workloads/).  With CWC_PARITY_OUT=<dir> each
config writes <dir>/parity_<config>.json (compared, matched, divergences by
class with the traced records): the committed report profiles/r02/parity.json
is assembled from those.
"""
import concurrent.futures as cf
import json
import multiprocessing as mp
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import workloads as w  # noqa: E402

from .tracer import first_sample_mismatch_t, trace_mismatches  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1010_2438_b200 import cwc  # noqa: E402

MIN_MATCH = 0.999
SUBSETS = [("C1", 1), ("C2", 8), ("C3", 16), ("C4", 32), ("C5", 32)]
TRACE_CAP = {"C1": 10_000, "C2": 400_000, "C3": 50_000, "C4": 80_000, "C5": 400_000}


def _oracle_chunk(args):
    name, g_chunk = args
    desc, sweep, cfg = w.config(name)
    r = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                        g_list=g_chunk, want_stats=False)
    return r["traj"], r["firings"], r["status"]


def oracle_subset(name, g_list):
    """The oracle on g_list, split over the host cores (order preserved)."""
    workers = max(1, min(os.cpu_count() or 1, 32))
    n_chunks = min(len(g_list), 4 * workers)
    chunks = [g_list[i::n_chunks] for i in range(n_chunks)]
    with cf.ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_oracle_chunk, [(name, c) for c in chunks]))
    J1, O = res[0][0].shape[1:]
    traj = np.zeros((len(g_list), J1, O), dtype=np.int64)
    fir = np.zeros(len(g_list), dtype=np.int64)
    st = np.zeros(len(g_list), dtype=np.int32)
    for i, (t, f, s) in enumerate(res):
        traj[i::n_chunks] = t
        fir[i::n_chunks] = f
        st[i::n_chunks] = s
    return traj, fir, st


@pytest.mark.parametrize("name,stride", SUBSETS, ids=[s[0] for s in SUBSETS])
def test_parity_at_survey_scale(name, stride):
    run_parity(name, stride)


def run_parity(name, stride, tag="parity"):
    desc, sweep, cfg = w.config(name)
    model = cwc.cwc_model_create(desc)
    R = cfg["n_replicas"]
    gpu = cwc.simulate(model, R, cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep, want_traj=True)
    bench_like = cwc.simulate(model, R, cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                              want_firings=False)  # the exact call bench.py times
    torch.cuda.synchronize()
    for k in ("count", "sum", "sumsq"):
        assert torch.equal(gpu[k], bench_like[k]), k
    P = gpu["n_points"]
    G = P * R
    # MM trajectories that convert all substrate stall legitimately (a0 = 0)
    assert np.isin(gpu["status"].cpu().numpy(), [cwc.CWC_TRAJ_DONE, cwc.CWC_TRAJ_STALLED]).all()
    # exact on-line moments == reduction of the kernel's own dump (every trajectory)
    t = gpu["traj"].view(P, R, gpu["traj"].shape[1], gpu["traj"].shape[2])
    assert int(t.abs().max().item()) ** 2 * R < 2**62
    assert (gpu["count"] == R).all()
    assert torch.equal(gpu["sum"], t.sum(dim=1))
    assert (gpu["sumsq"][..., 1] == 0).all()
    assert torch.equal(gpu["sumsq"][..., 0], (t * t).sum(dim=1))

    g_list = list(range(0, G, stride))
    del t
    t0 = time.time()
    o_traj, o_fir, o_st = oracle_subset(name, g_list)
    t_oracle = time.time() - t0
    idx = torch.as_tensor(np.asarray(g_list), device="cuda")
    g_traj = gpu["traj"][idx].cpu().numpy()
    g_fir = gpu["firings"][idx].cpu().numpy()
    g_st = gpu["status"][idx].cpu().numpy()
    same = (g_traj == o_traj).all(axis=(1, 2)) & (g_fir == o_fir) & (g_st == o_st)
    bad = [i for i in np.nonzero(~same)[0]]
    report = []
    if bad:
        report = trace_mismatches(model, desc, sweep, cfg, [g_list[i] for i in bad], cap=TRACE_CAP[name],
                                  gpu_rows=[g_traj[i] for i in bad], ora_rows=[o_traj[i] for i in bad])
    classes = {}
    for rec in report:
        classes[rec[1]] = classes.get(rec[1], 0) + 1
    out = {"config": name, "trajectories": G, "subset": "g = 0 mod %d" % stride, "compared": len(g_list),
           "matched": int(same.sum()), "match_fraction": float(same.mean()), "divergences_by_class": classes,
           "divergences": [{"g": r[0], "class": r[1], "record": r[2], "detail": r[3]} for r in report],
           "firings_compared": int(o_fir.sum()), "oracle_seconds": round(t_oracle, 1),
           "oracle_processes": max(1, min(os.cpu_count() or 1, 32)),
           "kernel_plan": "automatic (bench launch shape)"}
    dst = os.environ.get("CWC_PARITY_OUT")
    if dst:
        os.makedirs(dst, exist_ok=True)
        with open(os.path.join(dst, "%s_%s.json" % (tag, name)), "w") as f:
            json.dump(out, f, indent=1)
    for rec in report:
        assert rec[1] not in ("BUG", "identical-trace"), rec
    assert same.mean() >= MIN_MATCH, out
    # moments over the matched subset: mean / variance per sample time within 1e-9
    m = np.nonzero(same)[0]
    a = g_traj[m].astype(np.float64)
    b = o_traj[m].astype(np.float64)
    assert np.allclose(a.mean(axis=0), b.mean(axis=0), rtol=1e-9, atol=0)
    if len(m) > 1:
        assert np.allclose(a.var(axis=0, ddof=1), b.var(axis=0, ddof=1), rtol=1e-9, atol=1e-12)
