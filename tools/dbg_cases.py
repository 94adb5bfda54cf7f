import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as w
from paper_1010_2438_b200 import cwc
case = sys.argv[1]
if len(sys.argv) > 2:
    cwc.LIB_PATH = os.path.abspath(sys.argv[2])
cases = {
    "c1": (w.config("C1")[0], None, dict(t_end=100.0, sample_dt=1.0, n_replicas=1000)),
    "c3sweep": (w.config("C3")[0], w.mm_sweep(5, 7), dict(t_end=50.0, sample_dt=0.5, n_replicas=13)),
    "c3one": (w.config("C3")[0], None, dict(t_end=50.0, sample_dt=0.5, n_replicas=13)),
    "c3short": (w.config("C3")[0], w.mm_sweep(5, 7), dict(t_end=1.0, sample_dt=0.5, n_replicas=13)),
    "stall": (w.decay_model(3, 5.0), None, dict(t_end=10.0, sample_dt=1.0, n_replicas=65)),
    "dimer": (w.dimerisation_model(50, 0.1), None, dict(t_end=3.0, sample_dt=0.1, n_replicas=129)),
    "decay": (w.decay_model(1000, 1.0), None, dict(t_end=1.0, sample_dt=0.25, n_replicas=777)),
}
desc, sweep, cfg = cases[case]
model = cwc.cwc_model_create(desc)
print(case, "created", flush=True)
t0 = time.time()
out = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], 1, sweep=sweep, want_traj=True,
                   force_path=cwc.CWC_PATH_WARP)
torch.cuda.synchronize()
print(case, "ok %.2fs firings %d status %s" % (time.time() - t0, out["firings"].sum().item(), sorted(set(out["status"].tolist()))), flush=True)
