import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as w
from paper_1010_2438_b200 import cwc
cwc.LIB_PATH = os.path.abspath(sys.argv[1])
desc, sweep = w.config("C3")[0], w.mm_sweep(5, 7)
model = cwc.cwc_model_create(desc)
out = cwc.simulate(model, 13, 50.0, 0.5, 1, sweep=sweep, want_traj=True, force_path=cwc.CWC_PATH_WARP)
torch.cuda.synchronize()
print("firings", out["firings"].sum().item(), "status", out["status"].tolist()[:40])
