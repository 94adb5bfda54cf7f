"""Copy a round-end evidence run (gpurun_out/<tag>/, tools/gpu_final.sh) into
profiles/<round>/final/, regenerate profiles/ncu_bench.json (bench.py's
`traffic` source) and print the final-state table for profiles/README.md.

    python tools/profiles_final.py final2 [r02]
"""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r02"
src = os.path.join(ROOT, "gpurun_out", tag)
dst = os.path.join(ROOT, "profiles", rnd, "final")
shutil.rmtree(dst, ignore_errors=True)
os.makedirs(dst)
keep = re.compile(r"(bench_.*\.(json|err)|case_.*\.log|(no)?dumpcase_.*\.log|(no)?dump_dram_.*\.csv|gpu\.txt|launches\.csv|"
                  r"launch_plain\.json|ncu_full_summary\.json|ncu_summary\.log|pytest_gpu\.log|smoke\.log|lines_.*\.txt|"
                  r"parity_.*\.log)$")
for f in sorted(os.listdir(src)):
    p = os.path.join(src, f)
    if os.path.isdir(p) and f.startswith("parity_"):
        shutil.copytree(p, os.path.join(dst, f))
    elif keep.match(f):
        shutil.copy(p, dst)
summ = json.load(open(os.path.join(dst, "ncu_full_summary.json")))
bench_src = {}
for c, v in summ.items():
    v["report"] = "(not committed) gpurun_out/%s/full_%s.ncu-rep" % (tag, c)
    bench_src[c] = {"kernel": v["kernel"], "dram_bytes": v["dram_bytes"], "duration_ms": v["duration_ms"],
                    "source": "profiles/%s/final/ncu_full_summary.json: ncu --set full of the bench workload "
                              "(tools/run_case.py --config %s; C6: tools/dyn_probe.py 8192)" % (rnd, c)}
json.dump(summ, open(os.path.join(dst, "ncu_full_summary.json"), "w"), indent=1)
json.dump(bench_src, open(os.path.join(ROOT, "profiles", "ncu_bench.json"), "w"), indent=1)
print(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "profiles_table.py"), dst], capture_output=True,
                     text=True).stdout)
