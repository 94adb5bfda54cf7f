"""Two- vs four- vs eight-trajectories-per-warp kernels across network sizes (the
planner's crossover): random networks (workloads.random_network_model, the C4
generator at other sizes) and n-species Lotka-Volterra chains; firings/s by
kernel events, best of 3, with nvidia-smi clocks."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_1010_2438_b200 import cwc  # noqa: E402

if len(sys.argv) > 1:  # an experiment variant of the library (tools/build_variant.sh)
    cwc.LIB_PATH = os.path.abspath(sys.argv[1])
LIBTAG = os.path.basename(cwc.LIB_PATH)

cases = [("rnd", M, lambda M=M: wl.random_network_model(seed=1, n_species=64, n_reactions=M)) for M in (64, 96, 128, 160, 192, 224, 256)]
cases += [("lv", 129, lambda: wl.lotka_volterra_chain(128))]
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
ev[0].record()
ev[1].record()
for name, M, make in cases:
    model = cwc.cwc_model_create(make())
    t_end = 0.2 if name == "rnd" else 0.2
    for kname, kern in (("warp2", cwc.CWC_KERNEL_WARP2), ("warp8", cwc.CWC_KERNEL_WARP8), ("warp4", cwc.CWC_KERNEL_WARP4)):
        buf, best = None, None
        clk = ClockSampler(0)
        clk.start()
        for _ in range(3):
            out = cwc.simulate(model, 32768, t_end, 0.01, 1, force_path=cwc.CWC_PATH_WARP, kernel=kern, buffers=buf,
                               kernel_events=ev)
            torch.cuda.synchronize()
            buf = out
            ms = ev[0].elapsed_time(ev[1])
            best = ms if best is None else min(best, ms)
        c = clk.stop()
        f = float(out["firings"].double().sum())
        print(json.dumps({"lib": LIBTAG, "model": name, "M": model.info.n_reactions, "cells": model.info.n_cells, "kernel": kname,
                          "firings": f, "ms": best, "firings_per_s": f / best * 1e3, "clocks": c}), flush=True)
