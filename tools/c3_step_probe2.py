"""C3 step as bench.py runs it (prebuilt sweep arrays): GPU time before the
kernel vs the host's enqueue time of cwc_simulate, per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as w  # noqa: E402
from paper_1010_2438_b200 import cwc  # noqa: E402

desc, sweep, cfg = w.config("C3")
model = cwc.cwc_model_create(desc)
st = torch.cuda.current_stream()
R = cfg["n_replicas"]
J1 = int(cfg["t_end"] / cfg["sample_dt"]) + 1
P = len(sweep["values"])
ncell = P * J1 * model.info.n_obs
count = torch.empty(ncell, dtype=torch.int64, device="cuda")
s1 = torch.empty(ncell, dtype=torch.int64, device="cuda")
sq = torch.empty((ncell, 2), dtype=torch.int64, device="cuda")
ek = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for e in ek:
    e.record()
opts = cwc.cwc_sim_opts()
opts.force_path = cwc.CWC_PATH_AUTO
opts.ev_kernel_begin = ek[0].cuda_event
opts.ev_kernel_end = ek[1].cuda_event
ws = torch.empty(cwc.cwc_simulate_workspace_size(model, R, sweep, cfg["t_end"], cfg["sample_dt"], opts),
                 dtype=torch.uint8, device="cuda")
swa = cwc._SweepArrays(sweep)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(8):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    t0 = time.perf_counter()
    cwc.cwc_simulate(model, R, sweep, cfg["t_end"], cfg["sample_dt"], cfg["seed"], st.cuda_stream, (count, s1, sq), ws,
                     opts, sweep_arrays=swa)
    t1 = time.perf_counter()
    b.record(st)
    b.synchronize()
    print("step %.3f ms: before-kernel %.3f, kernel %.3f, after %.3f; host enqueue %.3f ms" % (
        a.elapsed_time(b), a.elapsed_time(ek[0]), ek[0].elapsed_time(ek[1]), ek[1].elapsed_time(b), (t1 - t0) * 1e3))
