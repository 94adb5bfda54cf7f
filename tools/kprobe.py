"""Kernel-time probe of one config (experiments; kernel events, best of 3):
    python tools/kprobe.py --config C2 [--t-end T] [--replicas R] [--kernel auto|ws|single|warp2|warp]
                           [--lib variant.so] [--tag name]
Prints one JSON line: firings/s, kernel ms, cycles per firing of the longest
trajectory at the SM clock (1965 MHz)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as w  # noqa: E402
from paper_1010_2438_b200 import cwc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--t-end", type=float, default=None)
ap.add_argument("--replicas", type=int, default=None)
ap.add_argument("--kernel", default="auto")
ap.add_argument("--lib", default=None)
ap.add_argument("--tag", default="")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--bps", type=int, default=0, help="blocks_per_sm override")
ap.add_argument("--wpb", type=int, default=0, help="warps_per_block override")
a = ap.parse_args()
if a.lib:
    cwc.LIB_PATH = os.path.abspath(a.lib)
K = {"auto": cwc.CWC_KERNEL_AUTO, "ws": cwc.CWC_KERNEL_THREAD_WS, "single": cwc.CWC_KERNEL_THREAD,
     "warp2": cwc.CWC_KERNEL_WARP2, "warp": cwc.CWC_KERNEL_WARP, "thread2": cwc.CWC_KERNEL_THREAD2,
     "ws2": cwc.CWC_KERNEL_THREAD_WS2, "warp8": cwc.CWC_KERNEL_WARP8, "warp4": cwc.CWC_KERNEL_WARP4}[a.kernel]
desc, sweep, cfg = w.config(a.config)
if a.t_end:
    cfg["t_end"] = a.t_end
if a.replicas:
    cfg["n_replicas"] = a.replicas
model = cwc.cwc_model_create(desc)
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
ev[0].record()
ev[1].record()
best, out, buf = None, None, None
for _ in range(a.reps):
    out = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                       kernel_events=ev, kernel=K, buffers=buf, blocks_per_sm=a.bps, warps_per_block=a.wpb)
    torch.cuda.synchronize()
    buf = out
    ms = ev[0].elapsed_time(ev[1])
    best = ms if best is None else min(best, ms)
f = out["firings"].double()
print(json.dumps({"tag": a.tag or os.path.basename(a.lib or "libcwcsim.so"), "config": a.config, "kernel": a.kernel,
                  "t_end": cfg["t_end"], "replicas": cfg["n_replicas"], "kernel_ms": best, "bps": a.bps, "wpb": a.wpb,
                  "firings": float(f.sum()), "firings_per_s": float(f.sum()) / best * 1e3,
                  "cycles_per_firing_max": best * 1e-3 * 1.965e9 / max(float(f.max()), 1.0)}), flush=True)
