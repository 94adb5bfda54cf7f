"""Run one cwc_simulate call on a config (profiling / ncu target).

    python tools/run_case.py --config C2 [--t-end 1.0] [--replicas N] [--path auto|thread|warp]
                             [--block-threads T] [--repeat K]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1010_2438_b200 import cwc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--t-end", type=float, default=None)
ap.add_argument("--replicas", type=int, default=None)
ap.add_argument("--path", default="auto", choices=["auto", "thread", "warp"])
ap.add_argument("--block-threads", type=int, default=0)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--dump", action="store_true", help="also write every trajectory sample (out_traj)")
a = ap.parse_args()
desc, sweep, cfg = wl.config(a.config)
if a.t_end:
    cfg["t_end"] = a.t_end
if a.replicas:
    cfg["n_replicas"] = a.replicas
model = cwc.cwc_model_create(desc)
path = {"auto": cwc.CWC_PATH_AUTO, "thread": cwc.CWC_PATH_THREAD, "warp": cwc.CWC_PATH_WARP}[a.path]
buf = None
for k in range(a.repeat):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                       force_path=path, block_threads=a.block_threads, buffers=buf, want_traj=a.dump)
    e1.record()
    torch.cuda.synchronize()
    buf = out
    f = int(out["firings"].sum().item())
    ms = e0.elapsed_time(e1)
    print("%s t_end=%g G=%d firings=%d ms=%.3f firings/s=%.4g" % (a.config, cfg["t_end"], out["firings"].numel(), f, ms,
                                                                 f / ms * 1e3), flush=True)
