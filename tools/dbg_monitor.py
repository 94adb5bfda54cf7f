"""Live progress monitor of the segment kernel (debug build with
-DCWC_WSEG_DEBUG -DCWC_DEBUG_KNOBS): per-segment state in host-mapped memory,
read while the kernel runs.  python tools/dbg_monitor.py LIB CASE"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import cuda.bindings.runtime as rt

import workloads as w
from paper_1010_2438_b200 import cwc

cwc.LIB_PATH = os.path.abspath(sys.argv[1])
case = sys.argv[2]
cases = {"decay": (w.decay_model(1000, 1.0), None, dict(t_end=1.0, sample_dt=0.25, n_replicas=int(os.environ.get("NREP", 777)))),
         "c1": (w.config("C1")[0], None, dict(t_end=100.0, sample_dt=1.0, n_replicas=64))}
desc, sweep, cfg = cases[case]
torch.zeros(1).cuda()
NB = 8 * 64 * 1024
err, hptr = rt.cudaHostAlloc(NB, rt.cudaHostAllocMapped)
err, dptr = rt.cudaHostGetDevicePointer(hptr, 0)
buf = (ctypes.c_uint64 * (NB // 8)).from_address(hptr)
ctypes.memset(hptr, 0, NB)
os.environ["CWC_PROF_PTR"] = str(int(dptr))
model = cwc.cwc_model_create(desc)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
  try:
    out = cwc.simulate(model, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], 1, sweep=sweep, want_traj=True,
                       force_path=cwc.CWC_PATH_WARP, stream=s.cuda_stream)
  except Exception as ex:
    print("simulate raised:", ex, flush=True)
for it in range(3):
    time.sleep(3)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8)
    bad = np.nonzero(a[:, 1] == 100)[0]
    for i in bad[:10]:
        r = a[i]
        print("BAD seg %d g %d mu %d hitsL %x posL %x L %d pos_any %x target %r a0 %r" % (i, r[2], np.int64(r[3]), r[4] >> 32, r[4] & 0xffffffff, r[5] & 0xffffffff, r[5] >> 32,
              np.frombuffer(r[6].tobytes(), np.float64)[0], np.frombuffer(r[7].tobytes(), np.float64)[0]), flush=True)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8)
    live = np.nonzero(a[:, 0])[0]
    print("t=%ds segments with progress: %d" % (3 * (it + 1), len(live)), flush=True)
    for i in live[:64]:
        r = a[i]
        print("seg %4d iter %12d code %d g %d n %d j %d kd %d flags %d a0 %r tn %r" % (
            i, r[0], r[1], r[2], r[3], r[4] >> 32, r[4] & 0xffffffff, r[5],
            np.frombuffer(r[6].tobytes(), np.float64)[0], np.frombuffer(r[7].tobytes(), np.float64)[0]), flush=True)
    if s.query():
        print("kernel finished")
        break
os._exit(0)
