"""Copy a round-end evidence run (gpurun_out/<tag>/, tools/gpu_final.sh) into
profiles/r01/<tag>/, regenerate profiles/ncu_bench.json (the `traffic` source
of bench.py) and the final-state table of profiles/README.md.

    python tools/profiles_update.py final6 [old_tag_to_remove]
"""
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out", tag)
dst = os.path.join(ROOT, "profiles", "r01", tag)
if len(sys.argv) > 2:
    shutil.rmtree(os.path.join(ROOT, "profiles", "r01", sys.argv[2]), ignore_errors=True)
os.makedirs(dst, exist_ok=True)
for f in os.listdir(src):
    if re.match(r"(bench_.*\.json|case_.*\.log|gpu\.txt|launches\.csv|ncu_full_summary\.json|pytest_gpu\.log|smoke\.log|lines_.*\.txt)$", f):
        shutil.copy(os.path.join(src, f), dst)

summ = json.load(open(os.path.join(dst, "ncu_full_summary.json")))
bench_src = {}
for c, v in summ.items():
    v["report"] = "(not committed) gpurun_out/%s/full_%s.ncu-rep" % (tag, c)
    bench_src[c] = {"kernel": v["kernel"], "dram_bytes": v["dram_bytes"], "duration_ms": v["duration_ms"],
                    "source": "profiles/r01/%s/ncu_full_summary.json: ncu --set full of tools/run_case.py --config %s "
                              "(the bench workload)" % (tag, c)}
json.dump(summ, open(os.path.join(dst, "ncu_full_summary.json"), "w"), indent=1)
json.dump(bench_src, open(os.path.join(ROOT, "profiles", "ncu_bench.json"), "w"), indent=1)

names = {"C1": "C1 immigration-death", "C2": "**C2 Lotka-Volterra (bench default)**", "C3": "C3 Michaelis-Menten sweep",
         "C4": "C4 random 64x256", "C5": "C5 CWC 1+32 compartments"}
rows = []
for c in ["C1", "C2", "C3", "C4", "C5"]:
    b = json.load(open(os.path.join(dst, "bench_%s.json" % c)))
    r = b["roofline"]
    n = summ[c]
    fir = int(re.search(r"firings=(\d+)", open(os.path.join(dst, "case_%s.log" % c)).read()).group(1))
    k = n["kernel"].split("(")[0].replace("void ", "")
    v, fr = "%.3g" % b["value"], "%.3f" % r["frac"]
    if c == "C2":
        v, fr = "**%s**" % v, "**%s**" % fr
    rows.append("| %s | %s | %s | %.2f | %s | %.3g | %.1f (floor %.1f) | %.1f %% | %.1f | %.1f %% | %.2g |" % (
        names[c], k, v, b["ms_per_step"], fr, b["e2e"]["value"], n["warp_inst"] / fir, r["ops_per_firing"] / 32,
        n["issue_active_pct"], n["threads_per_inst"], n["warps_active_pct"], n["dram_bytes"]))
ref = json.load(open(os.path.join(dst, "bench_reference.json")))
p = os.path.join(ROOT, "profiles", "README.md")
s = open(p).read()
i = s.index("## Round 1, final state")
j = s.index("(warp-inst per firing =")
s = s[:i] + """## Round 1, final state (`r01/%s/`)

| config | kernel (auto plan) | firings/s (`value`) | step ms | roofline frac (issue) | e2e firings/s | ncu: warp-inst per firing | issue active | threads/inst | warps active | DRAM bytes/launch |
|---|---|---|---|---|---|---|---|---|---|---|
%s

""" % (tag, "\n".join(rows)) + s[j:]
s = re.sub(r"\* Oracle \(CPU, single thread, the reference arm\): [0-9.e+]+ firings/s on C2",
           "* Oracle (CPU, single thread, the reference arm): %.3g firings/s on C2" % ref["value"], s)
open(p, "w").write(s)
print("\n".join(rows))
