"""GPU parity on EVERY trajectory of BASELINE's five full configs (the bench
launch shape) against the CPU oracle in a process pool over the host cores.
Opt-in (it takes ~10 minutes of oracle time on 16 cores): CWC_PARITY_FULL=1.
Same bar and tracer as tests/test_gpu_parity_scale.py; with CWC_PARITY_OUT
each config writes parity_full_<config>.json (the committed report
profiles/r02/parity_full.json is assembled from those)."""
import os

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
if os.environ.get("CWC_PARITY_FULL") != "1":
    pytest.skip("opt-in: CWC_PARITY_FULL=1", allow_module_level=True)

from .test_gpu_parity_scale import run_parity  # noqa: E402


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_parity_every_trajectory(name):
    run_parity(name, 1, tag="parity_full")
