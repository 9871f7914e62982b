"""Instruction/stall share of straight-line SASS blocks (runs of equal
execution count) of the first kernel in an ncu report; optional dump of a
SASS index range.  Usage: python tools/ncu_blocks.py REP [N] [A B]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iE] or 0) for r in data)
totW = sum(float(r[iW] or 0) for r in data) or 1
if len(sys.argv) > 3:
    for i in range(int(sys.argv[2]), int(sys.argv[3])):
        r = data[i]
        print(f"{i:6d} {float(r[iE] or 0) / tot * 100:5.2f}% w{float(r[iW] or 0) / totW * 100:5.1f}% {r[iS].strip()[:90]}")
    sys.exit()
blocks, cur = [], None
for i, r in enumerate(data):
    e = float(r[iE] or 0)
    if cur and e > 0 and abs(cur[2] - e) <= 0.5:
        cur[1] = i
        cur[3] += float(r[iW] or 0)
        cur[4] += 1
    else:
        if cur:
            blocks.append(cur)
        cur = [i, i, e, float(r[iW] or 0), 1]
blocks.append(cur)
print(f"total instructions {tot:.4g}, stall samples {totW:.4g}")
for b in sorted(blocks, key=lambda b: -b[2] * b[4])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"[{b[0]:5d}-{b[1]:5d}] n={b[4]:3d} exec={b[2]:.3e} share={b[2] * b[4] / tot * 100:5.1f}% "
          f"stall={b[3] / totW * 100:5.1f}%  {data[b[0]][iS].strip()[:48]}")
