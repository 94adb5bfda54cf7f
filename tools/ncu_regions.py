"""Stall reasons of SASS address regions of one kernel in an ncu report.

    python tools/ncu_regions.py report.ncu-rep name:start:end [name:start:end ...]
start/end are hex offsets from the kernel's first instruction.
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = list(csv.reader(out.splitlines()))
hdr = None
for i, r in enumerate(lines):
    if r and r[0] == "Address":
        hdr, start = r, i
        break
rows = [dict(zip(hdr, r)) for r in lines[start + 1:] if r]
base = int(rows[0]["Address"], 16)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows) or 1
for spec in sys.argv[2:]:
    name, a, b = spec.split(":")
    a, b = int(a, 16), int(b, 16)
    sel = [r for r in rows if a <= int(r["Address"], 16) - base < b]
    s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in sel)
    agg = {h: sum(int(r[h] or 0) for r in sel) for h in reasons}
    top = sorted(agg.items(), key=lambda kv: -kv[1])[:6]
    print("%-10s %5.1f%% of samples: %s" % (name, 100 * s / tot,
          ", ".join("%s %.0f%%" % (k[6:], 100 * v / max(s, 1)) for k, v in top)))
