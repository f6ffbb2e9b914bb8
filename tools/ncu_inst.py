"""Top source lines of one kernel by warp instructions executed.
    python tools/ncu_inst.py REP.ncu-rep KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, hdr, f = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    rows.append((inst, f"{f}:{r[0]}", r[1].strip()[:100]))
tot = sum(x[0] for x in rows) or 1
print(f"total warp instructions {tot}")
for i, l, s in sorted(rows, reverse=True)[:top]:
    print(f"{100 * i / tot:5.1f}% {i:10d} {l:22s} {s}")
