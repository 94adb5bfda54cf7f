import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import faulthandler
faulthandler.dump_traceback_later(15, exit=True)
import torch
import workloads as w
from paper_1010_2438_b200 import cwc
R = int(sys.argv[1]); variant = sys.argv[2]
kw = {}
if variant == "global": kw["stats_mode"] = cwc.CWC_STATS_GLOBAL
if variant == "seg32": kw["kernel"] = cwc.CWC_KERNEL_WARP
if variant == "bps1": kw["blocks_per_sm"] = 1
if variant == "nodump": pass
desc = w.decay_model(1000, 1.0)
model = cwc.cwc_model_create(desc)
print(R, variant, "created", flush=True)
t0 = time.time()
try:
    out = cwc.simulate(model, R, 1.0, 0.25, 1, want_traj=(variant != "nodump"), force_path=cwc.CWC_PATH_WARP, **kw)
    print("launched", flush=True)
    torch.cuda.synchronize()
    print(R, variant, "ok %.2fs firings %d" % (time.time() - t0, out["firings"].sum().item()), flush=True)
except Exception as ex:
    print(R, variant, "error", ex, flush=True)
