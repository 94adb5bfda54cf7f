"""NEXT-2: n-species Lotka-Volterra family, thread path vs warp paths.

    python tools/lv_family.py [--replicas 16384] [--t-end 1.0] [--out FILE]

For n in 2, 4, 8, 16, 32 (workloads.lotka_volterra_chain) runs every kernel
that can take the model -- the warp-specialised thread kernel (n <= 8 cells),
the two-trajectories-per-warp kernel (M <= 256) and the one-trajectory-per-warp
kernel -- and prints one JSON line per (n, kernel) with firings/s (CUDA
events around cwc_simulate, best of 3 after one warm-up).  The GPU analogue of
the paper's single-simulation SIMD study (fig:simd:speedup):
intra-trajectory data parallelism (lanes of a warp sharing one trajectory)
against inter-trajectory parallelism (one trajectory per lane).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from bench import ClockSampler  # noqa: E402  (nvidia-smi clocks during the timed runs)
from paper_1010_2438_b200 import cwc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--replicas", type=int, default=16384)
ap.add_argument("--t-end", type=float, default=1.0)
ap.add_argument("--out", default=None)
a = ap.parse_args()
lines = []
for n in (2, 4, 8, 16, 32, 64):
    model = cwc.cwc_model_create(wl.lotka_volterra_chain(n))
    kernels = []
    if model.info.thread_path_ok:
        kernels.append(("thread_ws", cwc.CWC_PATH_THREAD, cwc.CWC_KERNEL_THREAD_WS))
        kernels.append(("thread", cwc.CWC_PATH_THREAD, cwc.CWC_KERNEL_THREAD))
    if (model.info.n_reactions + 15) // 16 <= 16:
        kernels.append(("warp2", cwc.CWC_PATH_WARP, cwc.CWC_KERNEL_WARP2))
        kernels.append(("warp8", cwc.CWC_PATH_WARP, cwc.CWC_KERNEL_WARP8))
    kernels.append(("warp", cwc.CWC_PATH_WARP, cwc.CWC_KERNEL_WARP))
    for name, path, kern in kernels:
        clk = ClockSampler(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
        clk.start()
        best, buf = None, None
        for k in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = cwc.simulate(model, a.replicas, a.t_end, 0.01, 1, force_path=path, kernel=kern, buffers=buf)
            e1.record()
            torch.cuda.synchronize()
            buf = out
            ms = e0.elapsed_time(e1)
            if k > 0:
                best = ms if best is None else min(best, ms)
        clocks = clk.stop()
        f = int(out["firings"].sum().item())
        line = {"n_species": n, "reactions": model.info.n_reactions, "kernel": name, "replicas": a.replicas,
                "t_end": a.t_end, "firings": f, "ms": best, "firings_per_s": f / best * 1e3, "clocks": clocks}
        print(json.dumps(line), flush=True)
        lines.append(line)
if a.out:
    with open(a.out, "w") as fh:
        for line in lines:
            fh.write(json.dumps(line) + "\n")
