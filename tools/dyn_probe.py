"""Time the dynamic-topology kernel on the C6 workload (workloads/dynamic.py)."""
import json
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import workloads.dynamic as wd  # noqa: E402
from paper_1010_2438_b200 import cwc, cwc_dyn  # noqa: E402

if __import__("os").environ.get("CWC_PROBE_LIB"):  # an experiment variant (tools/build_variant.sh)
    cwc.LIB_PATH = __import__("os").path.abspath(__import__("os").environ["CWC_PROBE_LIB"])


def main():
    c = dict(wd.CONFIG_C6)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else c["n_replicas"]
    wpb = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    m = cwc_dyn.cwc_dyn_model_create(wd.cell_population_model())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    e1.record()  # torch creates the CUDA events on first record
    buf = None
    for it in range(4):
        r = cwc_dyn.simulate(m, n, c["t_end"], c["sample_dt"], c["seed"], kernel_events=(e0, e1), buffers=buf,
                             warps_per_block=wpb)
        buf = r["buffers"]
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        f = int(r["firings"].sum().item())
        st = torch.bincount(r["status"].long(), minlength=5).tolist()
        info = cwc_dyn.cwc_dyn_info_get(m, n, c["t_end"], c["sample_dt"])
        print(json.dumps(dict(n=n, ms=ms, firings=f, rate=f / ms * 1e3, status=st, blocks=info.blocks,
                              threads=info.threads, smem=info.smem_bytes)))


if __name__ == "__main__":
    main()
