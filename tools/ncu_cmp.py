"""Side-by-side of selected raw ncu metrics of several .ncu-rep captures
(first kernel of each).  Usage: python tools/ncu_cmp.py a.ncu-rep b.ncu-rep ..."""
import csv
import io
import re
import subprocess
import sys

PAT = re.compile(r"^(gpu__time_duration.sum|sm__cycles_elapsed.avg|smsp__issue_active.avg.pct_of_peak_sustained_active|"
                 r"sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed|"
                 r"sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active|"
                 r"smsp__inst_executed.sum|smsp__average_warps_issue_stalled_.*_per_issue_active.ratio|"
                 r"l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed|"
                 r"dram__bytes_read.sum|launch__registers_per_thread)$")


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, first = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, first) if PAT.match(h)}


caps = [load(p) for p in sys.argv[1:]]
keys = sorted(set().union(*caps))
for k in keys:
    vals = [c.get(k, ("", ""))[0] for c in caps]
    if all(v in ("", "0", "0.000000") for v in vals):
        continue
    print(f"{k:95s} " + " ".join(f"{v:>16s}" for v in vals))
