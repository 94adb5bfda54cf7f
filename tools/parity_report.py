"""Assemble profiles/r02/parity.json from the per-config reports the parity
tests write with CWC_PARITY_OUT (tools/gpu_final.sh: <out>/parity_scale/,
<out>/parity_full/, <out>/parity_dyn/).

    python tools/parity_report.py gpurun_out/<tag> profiles/r02/parity.json
"""
import glob
import json
import os
import sys

src, dst = sys.argv[1], sys.argv[2]


def load(sub):
    out = {}
    for f in sorted(glob.glob(os.path.join(src, sub, "parity_*.json"))):
        d = json.load(open(f))
        out[d.get("config", os.path.basename(f)[7:-5])] = d
    return out


rep = {
    "what": "GPU (automatic plan = the kernels bench.py times) vs the CPU oracle, same Philox streams; per trajectory: "
            "sampled observables at every sample time, firings and status compared bit for bit; every mismatch traced "
            "and classified by tests/tracer.py",
    "commands": [
        "CWC_PARITY_OUT=... pytest tests/test_gpu_parity_scale.py (GPUTEST, subsets of SURVEY 8(d))",
        "CWC_PARITY_FULL=1 CWC_PARITY_OUT=... pytest tests/test_gpu_parity_full.py (every trajectory)",
        "CWC_PARITY_OUT=... pytest tests/test_gpu_dynamic.py -k survey (C6, dynamic topology, g = 0 mod 16)",
    ],
    "hardware": "1x NVIDIA B200 (148 SMs); oracle: host cores (process pool)",
    "source": src,
    "subsets": load("parity_scale"),
    "every_trajectory": load("parity_full"),
    "dynamic_topology": load("parity_dyn"),
}
tot = dict(trajectories_compared=0, matched=0, firings_compared=0, divergences=0)
for part in ("every_trajectory", "dynamic_topology"):
    for d in rep[part].values():
        tot["trajectories_compared"] += int(d.get("compared", 0))
        tot["matched"] += int(d.get("matched", 0))
        tot["firings_compared"] += int(d.get("firings_compared", 0))
        tot["divergences"] += len(d.get("divergences", d.get("divergent", [])))
rep["summary"] = tot
json.dump(rep, open(dst, "w"), indent=1)
print(json.dumps(tot))
