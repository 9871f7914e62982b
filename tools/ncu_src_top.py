"""Top stall lines and stall reasons of an ncu report's SASS source page (development tool)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
iA, iS = h.index("Address"), h.index("Source")
iW, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(r[iW] or 0) for r in data)
totE = sum(float(r[iE] or 0) for r in data)
print(rows[0][1][:70], "samples", tot, "instr", totE)
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.Counter()
for r in data:
    for c in cols:
        agg[c] += float(r[h.index(c)] or 0)
print([(k, round(v / tot * 100, 1)) for k, v in agg.most_common(6)])
for r in sorted(data, key=lambda r: -float(r[iW] or 0))[:n]:
    print(f"{r[iA][-5:]} {float(r[iW]) / tot * 100:5.1f}% exec={r[iE]:>8s} {r[iS][:80]}")
