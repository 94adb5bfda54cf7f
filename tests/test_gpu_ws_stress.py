"""Race stress test of the warp-specialised thread kernel's producer/consumer
hand-off (stands in for compute-sanitizer racecheck/synccheck, closed on this
GPU pool).  A test build with -DCWC_WS_STRESS=1 shrinks the draw ring to the
smallest legal size (8 draws per trajectory: the producer is at most one
round ahead, so every slot is reused constantly) and injects pseudo-random
sleeps of up to ~4 us between the producer's slot writes and its release
store and between the consumer's slot reads and its release store, per lane.
Any ordering bug of the hand-off (a slot overwritten before it was read, a
slot read before it was written) then corrupts draws and changes results.
The stressed kernel must reproduce the single-warp kernel of the normal
build (which has no hand-off at all) bit for bit -- moments, firings,
statuses -- across seeds and grid sizes (one CTA to several waves)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import workloads as w  # noqa: E402
from paper_1010_2438_b200 import _build, cwc  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("C2", 32, 0.2, 3), ("C2", 4000, 0.05, 5), ("C2", 40000, 0.02, 7), ("C1", 1024, 20.0, 1), ("C3", 48, 5.0, 2)]

CHILD = r'''
import json, os, sys
sys.path.insert(0, %r)
import numpy as np
import torch
import workloads as w
from paper_1010_2438_b200 import cwc
cwc.LIB_PATH = %r
out = {}
for name, R, T, seed in %r:
    desc, sweep, cfg = w.config(name)
    if sweep is not None:
        sweep = w.mm_sweep(6, 6)
    m = cwc.cwc_model_create(desc)
    r = cwc.simulate(m, R, T, cfg["sample_dt"], seed, sweep=sweep, kernel=cwc.CWC_KERNEL_THREAD_WS)
    torch.cuda.synchronize()
    key = "%%s_%%d_%%d" %% (name, R, seed)
    np.savez(os.path.join(%r, key + ".npz"), **{k: r[k].cpu().numpy() for k in ("count", "sum", "sumsq", "firings", "status")})
print("ok")
'''


@pytest.fixture(scope="module")
def stress_lib():
    env = dict(os.environ, CWC_BUILD_TAG="stress", NVCC_EXTRA="-DCWC_WS_STRESS=1")
    r = subprocess.run([sys.executable, "-c", "from paper_1010_2438_b200 import _build; print(_build.build())"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


def test_ws_handoff_under_stress_equals_single_warp_kernel(stress_lib, tmp_path):
    child = CHILD % (ROOT, stress_lib, CASES, str(tmp_path))
    r = subprocess.run([sys.executable, "-c", child], cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
    for name, R, T, seed in CASES:
        desc, sweep, cfg = w.config(name)
        if sweep is not None:
            sweep = w.mm_sweep(6, 6)
        ref = cwc.simulate(cwc.cwc_model_create(desc), R, T, cfg["sample_dt"], seed, sweep=sweep,
                           kernel=cwc.CWC_KERNEL_THREAD)
        torch.cuda.synchronize()
        got = np.load(tmp_path / ("%s_%d_%d.npz" % (name, R, seed)))
        for k in ("count", "sum", "sumsq", "firings", "status"):
            assert np.array_equal(got[k], ref[k].cpu().numpy()), (name, R, seed, k)
