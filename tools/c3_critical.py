"""C3 critical-path probe: time the longest sweep points alone (a few lone
warps) against the full sweep, one-shot kernel, kernel-event timing."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as w  # noqa: E402
from paper_1010_2438_b200 import cwc  # noqa: E402

desc, sweep, cfg = w.config("C3")
model = cwc.cwc_model_create(desc)
R, T, dt = cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"]


KERNEL = cwc.CWC_KERNEL_AUTO


def timed(sw, reps=R):
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev[0].record()
    ev[1].record()
    out = None
    ms = []
    for _ in range(3):
        out = cwc.simulate(model, reps, T, dt, 1, sweep=sw, kernel_events=ev, kernel=KERNEL)
        torch.cuda.synchronize()
        ms.append(ev[0].elapsed_time(ev[1]))
    return min(ms), out


full_ms, full = timed(sweep)
fir = full["firings"].view(-1, R).double().mean(dim=1).cpu().numpy()
order = np.argsort(-fir)
print(json.dumps(dict(case="full", kernel_ms=full_ms, max_point_firings=float(fir.max()),
                      mean_point_firings=float(fir.mean()))))
for k in (1, 2, 8, 32, 128, 512):
    sub = {"rules": sweep["rules"], "values": [sweep["values"][i] for i in order[:k]]}
    ms, out = timed(sub)
    f = int(out["firings"].max())
    print(json.dumps(dict(case="top%d" % k, points=k, kernel_ms=ms, max_firings=f, ns_per_firing=ms * 1e6 / f)))

if os.environ.get("WS_TOO"):
    KERNEL = cwc.CWC_KERNEL_THREAD_WS
    for k in (8, 128, 512, 1024, 4096):
        sub = {"rules": sweep["rules"], "values": [sweep["values"][i] for i in order[:k]]}
        ms, out = timed(sub)
        f = int(out["firings"].max())
        print(json.dumps(dict(case="ws_top%d" % k, points=k, kernel_ms=ms, max_firings=f, ns_per_firing=ms * 1e6 / f)))
    KERNEL = cwc.CWC_KERNEL_THREAD
    for k in (1024, 4096):
        sub = {"rules": sweep["rules"], "values": [sweep["values"][i] for i in order[:k]]}
        ms, out = timed(sub)
        print(json.dumps(dict(case="st_top%d" % k, points=k, kernel_ms=ms)))
