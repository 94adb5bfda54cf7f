"""Cycle accounting of the warp-specialised consumer (debug hook CWC_PROF_PTR).

Needs a library built with the accounting compiled in:
    NVCC_EXTRA=-DCWC_WS_PROF=1 python -c "from paper_1010_2438_b200 import _build; _build.build(force=True)"
    python tools/ws_prof.py --config C2 [--t-end 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1010_2438_b200 import cwc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--t-end", type=float, default=None)
ap.add_argument("--replicas", type=int, default=None)
ap.add_argument("--lib", default=None, help="variant library (tools/build_variant.sh)")
a = ap.parse_args()
if a.lib:
    cwc.LIB_PATH = os.path.abspath(a.lib)
desc, sweep, cfg = wl.config(a.config)
if a.t_end:
    cfg["t_end"] = a.t_end
if a.replicas:
    cfg["n_replicas"] = a.replicas
model = cwc.cwc_model_create(desc)
buf = torch.zeros(8, dtype=torch.int64, device="cuda")
os.environ["CWC_PROF_PTR"] = str(buf.data_ptr())
out = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                   kernel=cwc.CWC_KERNEL_THREAD_WS)
torch.cuda.synchronize()
v = buf.cpu().tolist()
nb = max(v[4], 1)
print("warps*batches %d  cycles/batch: wait %.0f fast %.0f records %.0f exact %.0f  | total/batch %.0f" % (
    nb, v[0] / nb, v[1] / nb, v[2] / nb, v[3] / nb, v[5] / nb))
