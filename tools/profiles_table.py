"""Markdown table of a round-end evidence directory (bench lines + ncu
summaries): python tools/profiles_table.py profiles/r02/final"""
import json
import os
import sys

d = sys.argv[1]
summ = json.load(open(os.path.join(d, "ncu_full_summary.json")))
names = {"C1": "C1 immigration-death", "C2": "**C2 Lotka-Volterra (bench default)**", "C3": "C3 Michaelis-Menten sweep",
         "C4": "C4 random 64x256", "C5": "C5 CWC 1+32 compartments", "C6": "C6 dynamic CWC cell population (NEXT-4)"}
print("| config | kernel (auto plan) | firings/s (`value`) | step ms | roofline frac (issue) | e2e firings/s | ncu: warp-inst per firing | issue active | threads/inst | warps active | DRAM bytes/launch |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for c in ("C1", "C2", "C3", "C4", "C5", "C6"):
    f = os.path.join(d, "bench_%s.json" % c)
    if not os.path.exists(f):
        continue
    b = json.loads(open(f).read().strip().splitlines()[-1])
    s = summ.get(c, {})
    kern = s.get("kernel", b["roofline"]["kernel"]).replace("void ", "").split("(")[0]
    wi = s.get("warp_inst", 0.0) / max(b["firings_per_step"], 1) if s else float("nan")
    # ncu captures the same workload as the bench step (C6: tools/dyn_probe.py at 8192 replicas)
    bold = c == "C2"
    v = "**%.3g**" % b["value"] if bold else "%.3g" % b["value"]
    fr = "**%.3f**" % b["roofline"]["frac"] if bold else "%.3f" % b["roofline"]["frac"]
    print("| %s | %s | %s | %.2f | %s | %.3g | %.1f | %.1f %% | %.1f | %.1f %% | %.2g |" % (
        names[c], kern, v, b["ms_per_step"], fr, b["e2e"]["value"], wi, s.get("issue_active_pct", 0),
        s.get("threads_per_inst", 0), s.get("warps_active_pct", 0), s.get("dram_bytes", 0)))
