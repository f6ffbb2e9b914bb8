"""Print duration / instructions / SM-active spread of kernels in an ncu report.

    python tools/ncu_quick.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__cycles_active.avg",
           "l1tex__cycles_active.max", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for row in rows[2:]:
    d = dict(zip(h, row))
    print(f"{d['Kernel Name'][:36]:36s} " + " ".join(f"{m.split('.')[0].split('__')[1][:14]}={d.get(m, '?')}"
                                                   for m in METRICS))
