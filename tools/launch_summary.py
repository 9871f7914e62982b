"""Summarise an ncu --metrics gpu__time_duration.sum launch list (last encode)."""
import collections
import csv
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1 / 3
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
data = rows[1:]
tail = data[int(len(data) * (1 - frac)):]
agg = collections.OrderedDict()
tot = 0.0
for r in tail:
    name = r[ik].split("(")[0].replace("void ", "")[-60:]
    v = float(r[iv].replace(",", "")) / 1000
    agg.setdefault(name, [0, 0.0])
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"launches {len(tail)} total {tot:.1f} us")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v:9.1f} us {100 * v / tot:5.1f}% {c:4d}x  {k}")
