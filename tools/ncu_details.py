"""Compact per-kernel view of an ncu report's details page.

    python tools/ncu_details.py REP.ncu-rep [regex-on-kernel] [metric-substring ...]
"""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
kre = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
want = sys.argv[3:] or ["Duration", "Memory Throughput", "Achieved Occupancy", "Registers Per Thread",
                        "Warp Cycles Per Issued Instruction", "Issue Slots Busy", "Block Limit Registers",
                        "Block Limit Shared Mem", "L1/TEX Hit Rate", "L2 Hit Rate", "Theoretical Occupancy",
                        "DRAM Throughput", "Eligible Warps Per Scheduler"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
iK, iS, iN, iU, iV = (hdr.index(c) for c in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
iID = hdr.index("ID")
seen = {}
for r in rows[1:]:
    if len(r) <= iV:
        continue
    k = r[iK].split("(")[0].replace("void ", "")
    if kre and not kre.search(k):
        continue
    key = (r[iID], k)
    for w in want:
        if r[iN] == w:
            seen.setdefault(key, []).append(f"{w}={r[iV]}{r[iU]}")
for (i, k), v in seen.items():
    print(f"[{i}] {k}\n    " + "\n    ".join(v))
