"""Per-launch DRAM traffic of an ncu --set full report -> profiles JSON (bench roofline.traffic)."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[0]
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6,
         "msecond": 1e-3, "second": 1.0}
ir, iw, it = (h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"),
              h.index("gpu__time_duration.sum"))
launches = []
for k, r in enumerate(rows[2:]):
    f = lambda i: float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
    launches.append(dict(launch=k, duration_s=f(it), dram_read_bytes=f(ir), dram_write_bytes=f(iw)))
json.dump(dict(source=sys.argv[3] if len(sys.argv) > 3 else rep, launches=launches), open(out, "w"),
          indent=1)
print(json.dumps(launches, indent=1))
