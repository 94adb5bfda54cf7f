"""Where the C3 step's non-kernel time goes: events around each enqueued
operation of cwc_simulate (host staging, memsets, kernel, stage 2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as w  # noqa: E402
from paper_1010_2438_b200 import cwc  # noqa: E402

desc, sweep, cfg = w.config("C3")
model = cwc.cwc_model_create(desc)
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for e in ev:
    e.record()  # torch creates the CUDA event at the first record; the library re-records them
buf = None
for it in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    out = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                       kernel_events=(ev[0], ev[1]), buffers=buf)
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    buf = out
    print("step %.3f ms: before-kernel %.3f, kernel %.3f, after-kernel %.3f; host enqueue %.3f ms" % (
        a.elapsed_time(b), a.elapsed_time(ev[0]), ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(b), (t1 - t0) * 1e3))
