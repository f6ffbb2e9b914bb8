"""Top source lines of one kernel in an ncu report by stall samples and
instructions executed (CUDA source view with SASS correlation).

    python tools/ncu_lines.py REP.ncu-rep KERNEL_REGEX [N]
"""
import csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = []
cur_file = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        stall = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    rows.append((stall, inst, f"{cur_file}:{r[0]}", r[1].strip()[:110]))
tot_s = sum(x[0] for x in rows) or 1
tot_i = sum(x[1] for x in rows) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for s, i, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% stall {100*i/tot_i:5.1f}% inst  {loc:18s} {src}")
