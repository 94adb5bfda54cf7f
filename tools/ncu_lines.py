"""Per-CUDA-source-line instruction / stall summary of an ncu report.

    python tools/ncu_lines.py report.ncu-rep [top]
Reads `ncu -i --page source --csv --print-source cuda,sass` and prints the
source lines with the most executed warp instructions and stall samples.
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = None
rows = []
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        ie = int(d["Instructions Executed"])
        st = int(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    rows.append((ie, st, fname, r[0], r[1].strip()[:90]))
tot_i = sum(x[0] for x in rows) or 1
tot_s = sum(x[1] for x in rows) or 1
print("total warp inst %d, stall samples %d" % (tot_i, tot_s))
for ie, st, f, ln, src in sorted(rows, key=lambda x: -x[1])[:top]:
    print("%5.1f%% inst %5.1f%% samples  %s:%s  %s" % (100 * ie / tot_i, 100 * st / tot_s, f, ln, src))
