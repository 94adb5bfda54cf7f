"""NEXT-1 study: cost / benefit of resumable runs (firing quanta with live-list
compaction, sample windows) against the one-shot kernel, full BASELINE
configs on one GPU.  Prints one JSON line per (config, schedule):
wall ms of the whole run (all advances, host syncs included), the sum of the
SSA kernels' event times, advances, firings/s.

    python tools/resume_study.py [C3 C2 ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as w  # noqa: E402
from bench import ClockSampler  # noqa: E402  (nvidia-smi clocks during the timed runs)
from paper_1010_2438_b200 import cwc  # noqa: E402

SCHEDULES = {
    "C2": [dict(quantum=0), dict(windows=[251, 501, 751, 1001]), dict(quantum=20000), dict(quantum=60000)],
    "C3": [dict(quantum=0), dict(quantum=1000), dict(quantum=2000), dict(quantum=4000), dict(quantum=8000),
           dict(windows=[26, 51, 76, 101])],
    "C4": [dict(quantum=0), dict(windows=[26, 51, 76, 101]), dict(quantum=10000)],
    "C5": [dict(quantum=0), dict(windows=[51, 101, 151, 201]), dict(quantum=100000)],
}


def run(name):
    desc, sweep, cfg = w.config(name)
    model = cwc.cwc_model_create(desc)
    R, T, dt = cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"]
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev[0].record()  # torch must see them recorded once; the library re-records them around each kernel
    ev[1].record()
    # one-shot reference
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        one = cwc.simulate(model, R, T, dt, 1, sweep=sweep)
        b.record()
        torch.cuda.synchronize()
    fir = int(one["firings"].sum())
    ms = a.elapsed_time(b)
    print(json.dumps(dict(config=name, schedule="one-shot", ms=round(ms, 3), firings_per_s=fir / ms * 1e3)), flush=True)
    for sch in SCHEDULES[name]:
        clk = ClockSampler(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
        clk.start()
        kern = [0.0]

        def ck(state, k):
            kern[0] += ev[0].elapsed_time(ev[1])
            return None

        for _ in range(2):
            kern[0] = 0.0
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            res = cwc.simulate_resumable(model, R, T, dt, 1, sweep=sweep, kernel_events=ev, checkpoint=ck, **sch)
            b.record()
            torch.cuda.synchronize()
        clocks = clk.stop()
        same = all(torch.equal(one[k], res[k]) for k in ("count", "sum", "sumsq", "firings", "status"))
        ms = a.elapsed_time(b)
        print(json.dumps(dict(config=name, schedule=sch, ms=round(ms, 3), kernel_ms=round(kern[0], 3),
                              advances=res["advances"], firings_per_s=fir / ms * 1e3, identical=same,
                              clocks=clocks)), flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or ["C3", "C2", "C4", "C5"]):
        run(n)
