"""C2 latency probe: cycles per firing of one trajectory (kernel-event time x
SM clock / firings per trajectory) as the number of CTAs grows, for the
warp-specialised and the single-warp thread kernels.  One lone CTA shows the
dependent-chain latency; the full run adds sub-partition sharing."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as w  # noqa: E402
from paper_1010_2438_b200 import cwc  # noqa: E402

if os.environ.get("PROBE_LIB"):
    cwc.LIB_PATH = os.path.abspath(os.environ["PROBE_LIB"])
desc, sweep, cfg = w.config("C2")
model = cwc.cwc_model_create(desc)
T = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
ev[0].record()
ev[1].record()
for kern, kname in ((cwc.CWC_KERNEL_THREAD_WS, "ws"), (cwc.CWC_KERNEL_THREAD, "single")):
    for R in [int(x) for x in os.environ.get("PROBE_R", "32,2368,4736,9472,14208,16384,18944").split(",")]:
        best = None
        for _ in range(3):
            out = cwc.simulate(model, R, T, cfg["sample_dt"], 1, kernel_events=ev, kernel=kern)
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1])
            best = ms if best is None else min(best, ms)
        f = out["firings"].double()
        per = float(f.mean())
        print(json.dumps({"kernel": kname, "replicas": R, "ctas": R // 32, "kernel_ms": best,
                          "firings_per_traj": per, "cycles_per_firing": best * 1e-3 * 1.965e9 / float(f.max()),
                          "firings_per_s": float(f.sum()) / best * 1e3}), flush=True)
