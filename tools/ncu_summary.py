#!/usr/bin/env python
"""Summarise an ncu report into per-kernel rows and per-entry-point DRAM
traffic (what bench.py reports as roofline.traffic).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_traffic.json

Reads `ncu -i REP --page raw --csv` (ncu is available without a GPU).  Each
C-ABI entry point maps to the kernels it launches; traffic per call is the
sum of dram__bytes_read.sum + dram__bytes_write.sum over one launch of each.
"""

from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size"]

# entry point -> kernel-name regexes (one launch each per call)
ENTRY_KERNELS = {
    "sf_quantize": [r"k_quant8_vec"],
    "sf_dequant8": [r"k_dequant8_vec"],
    "sf_prescale_exp": [r"k_prescale_hist<(0|false), (0|false)>", r"k_prescale_exact", r"k_prescale_refine"],
    "sf_gelu_fwd_prescale": [r"k_prescale_hist<(1|true), (0|false)>", r"k_prescale_exact", r"k_prescale_refine"],
    "sf_quant4_pack": [r"k_pack4_vec"],
    "sf_unpack4_dequant": [r"k_unpack4_vec"],
    "sf_prune_topk": [r"k_prune<(1|true), (0|false)>"],
    "sf_prune_topk_hint": [r"k_prune<(1|true), (1|true)>"],
    "sf_restore": [r"k_restore\b"],
    "sf_layernorm_fwd": [r"k_ln_fwd"],
    "sf_layernorm_bwd": [r"k_ln_bwd_lean<\d+, 1>"],
    "sf_gelu_bwd_packed4": [r"k_gelu_bwd_p4"],
    "sf_softmax_fwd_q8": [r"k_softmax_fwd_q8"],
    "sf_softmax_bwd_q8": [r"k_softmax_bwd_q8"],
    "sf_layer_distance": [r"k_dist_chunks<1>", r"k_dist_layers"],
    "sf_gelu_fwd_prescale_bias": [r"k_prescale_hist<(1|true), (1|true)>", r"k_prescale_exact",
                                  r"k_prescale_refine"],
    "sf_layernorm_fwd_residual": [r"k_ln_fwd<\d+, (1|true)>"],
    "sf_split_heads": [r"k_split_heads<(1|true), (0|false)>"],
    "sf_merge_heads": [r"k_merge_heads"],
    "sf_attention_fwd": [r"k_attn_fwd_tc5h\b"],
    "sf_attention_bwd": [r"k_attn_bwd_tc5h\b"],
    "sf_split3_bf16": [r"k_split3_flat"],
    "sf_split3_bf16_t": [r"k_split3_t\b"],
    "sf_gemm_split6": [r"k_gemm_split6_persistent<\d+, 3"],
    "sf_gemm_f16x3": [r"k_gemm_split6_persistent<\d+, 2"],
    "sf_split2_f16": [r"k_split2h_flat"],
    "sf_restore_rows": [r"k_restore_rows"],
}


# element (or parameter) count per call in paper_2305_18513_b200/kernel_bench.py
# at BERT-base B=128, T=128 (what the captured launches processed)
_BT4H, _BTH, _BHTT = 128 * 128 * 3072, 128 * 128 * 768, 128 * 12 * 128 * 128
BENCH_N = {"sf_quantize": _BT4H, "sf_dequant8": _BT4H, "sf_prescale_exp": _BT4H,
           "sf_gelu_fwd_prescale": _BT4H, "sf_quant4_pack": _BT4H, "sf_unpack4_dequant": _BT4H,
           "sf_gelu_bwd_packed4": _BT4H, "sf_softmax_fwd_q8": _BHTT, "sf_softmax_bwd_q8": _BHTT,
           "sf_prune_topk": _BTH, "sf_prune_topk_hint": _BTH, "sf_restore": _BTH, "sf_layernorm_fwd": _BTH,
           "sf_layernorm_bwd": _BTH, "sf_layer_distance": 768 * 3072 * 2 + 3072 + 768 + 30522 * 768,
           "sf_gelu_fwd_prescale_bias": _BT4H, "sf_layernorm_fwd_residual": _BTH, "sf_split_heads": _BTH,
           "sf_merge_heads": _BTH, "sf_attention_fwd": 128 * 12, "sf_attention_bwd": 128 * 12,
           "sf_split3_bf16": _BT4H, "sf_split3_bf16_t": _BT4H, "sf_split2_f16": _BT4H, "sf_restore_rows": _BTH}


def rows(rep: str):
    if rep.endswith(".csv"):          # a saved `--page raw --csv` export
        out = open(rep).read()
        out = out[out.index('"ID"'):]
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                             capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    idx = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,          # -> bytes
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}  # -> microseconds
    res = []
    for row in r[2:]:
        d = {"kernel": row[idx["Kernel Name"]]}
        for m in METRICS:
            if m not in idx:
                d[m] = None
                continue
            v = row[idx[m]].replace(",", "")
            try:
                d[m] = float(v) * scale.get(units[idx[m]], 1.0)
            except ValueError:
                d[m] = None
        res.append(d)
    return res


def summarise(rep: str):
    rs = rows(rep)
    per_kernel = defaultdict(list)
    for r in rs:
        per_kernel[r["kernel"]].append(r)
    kernels = {}
    for k, lst in per_kernel.items():
        n = len(lst)
        kernels[k] = {m: sum((x[m] or 0.0) for x in lst) / n for m in METRICS}
        kernels[k]["launches"] = n
    entries = {}
    for e, pats in ENTRY_KERNELS.items():
        tot_b, tot_t, found = 0.0, 0.0, []
        for i, pat in enumerate(pats):
            hit = [k for k in kernels if re.search(pat, k)]
            if not hit:
                if i == 0:            # the entry's main kernel was not captured
                    break
                continue
            k = hit[0]
            found.append(k.split("(")[0])
            tot_b += kernels[k]["dram__bytes_read.sum"] + kernels[k]["dram__bytes_write.sum"]
            tot_t += kernels[k]["gpu__time_duration.sum"]
        if found:
            n = BENCH_N.get(e)
            entries[e] = {"dram_bytes_per_call": tot_b, "ncu_us_per_call": tot_t, "kernels": found,
                          "n": n, "dram_bytes_per_elt": tot_b / n if n else None}
    return kernels, entries


if __name__ == "__main__":
    rep, out = sys.argv[1], sys.argv[2]
    kernels, entries = summarise(rep)
    json.dump({"report": rep, "entries": entries,
               "kernels": {k.split("(")[0]: v for k, v in kernels.items()}}, open(out, "w"), indent=1)
    for e, v in entries.items():
        print(f"{e:24s} {v['dram_bytes_per_call'] / 1e6:10.2f} MB  {v['kernels']}")
