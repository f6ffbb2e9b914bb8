#!/usr/bin/env python
"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file L.csv python bench.py ...`) into per-kernel totals and shares.

    python tools/launch_summary.py gpurun_out/launches.csv [out.txt]

ncu serialises launches and runs them cold, so the absolute times are
pessimistic; the shares are what the bench's kernel table must agree with.
"""
import csv
import io
import re
import sys
from collections import defaultdict


def load(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    out = []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        out.append((r["Kernel Name"], us))
    return out


def family(name):
    if "sf::" in name:
        return re.sub(r"\(.*", "", name).replace("void ", "")
    if "gemm" in name.lower() or "sgemm" in name.lower() or "cutlass" in name.lower():
        return "cuBLAS GEMM"
    return "torch elementwise/reduce"


def main():
    launches = load(sys.argv[1])
    tot = sum(t for _, t in launches)
    fam = defaultdict(lambda: [0, 0.0])
    for n, t in launches:
        f = fam[family(n)]
        f[0] += 1
        f[1] += t
    lines = [f"{len(launches)} launches, {tot / 1e3:.2f} ms total (ncu: serialised, cold caches)",
             f"{'kernel':48s} {'launches':>8s} {'ms':>9s} {'share':>7s}"]
    for k, (c, t) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:48]:48s} {c:8d} {t / 1e3:9.3f} {t / tot:7.2%}")
    ours = sum(t for k, (c, t) in fam.items() if k.startswith("sf::"))
    lines.append(f"own sf:: kernels: {ours / tot:.2%} of GPU time")
    txt = "\n".join(lines)
    print(txt)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt + "\n")


if __name__ == "__main__":
    main()
