"""Static schedule of a SASS region: sum of the per-instruction stall
counts (control bits 105..108) between two instruction addresses.

    cuobjdump -sass -fun <kernel> lib.cubin > k.sass
    python tools/sass_sched.py k.sass <start_hex> <end_hex>
"""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
ins = []
i = 0
while i < len(lines):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", lines[i])
    if m and i + 1 < len(lines):
        m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        addr = int(m.group(1), 16)
        hiw = int(m2.group(1), 16)
        stall = (hiw >> 41) & 0xF
        waitm = (hiw >> 52) & 0x3F
        ins.append((addr, m.group(2).strip(), stall, waitm))
        i += 2
        continue
    i += 1
sel = [x for x in ins if lo <= x[0] < hi]
tot = sum(x[2] for x in sel)
waits = sum(1 for x in sel if x[3])
print("instructions %d, static stall cycles %d (%.2f / inst), instructions with scoreboard waits %d" % (
    len(sel), tot, tot / max(1, len(sel)), waits))
ops = {}
for x in sel:
    op = re.sub(r"^@!?U?P\w+\s+", "", x[1]).split()[0].split(".")[0]
    ops.setdefault(op, [0, 0])
    ops[op][0] += 1
    ops[op][1] += x[2]
for op, (n, s) in sorted(ops.items(), key=lambda kv: -kv[1][1])[:15]:
    print("  %-8s n=%4d stall=%5d" % (op, n, s))
