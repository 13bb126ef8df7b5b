#!/usr/bin/env python3
"""Summarise the ncu A/B captures (gpurun_out/ncu_ab_<cfg>_<dmma|dfma>.csv) into a markdown table."""
import csv
import glob
import os
import sys

KEYS = [("gpu__time_duration.sum", "time (us)", 1e-3),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor (DMMA) pipe %", 1),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 (DFMA) pipe %", 1),
        ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue active %", 1),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts / CTA", None),
        ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-inst / CTA", None)]


def load(path):
    out = {}
    lines = [ln for ln in open(path) if ln.startswith('"')]
    for r in csv.DictReader(lines):
        out["kernel"] = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        out["grid"] = int(r["Grid Size"].strip("()").split(",")[0])
        out[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return out


def main(src="gpurun_out"):
    rows = []
    for p in sorted(glob.glob(os.path.join(src, "ncu_ab_*.csv"))):
        tag = os.path.basename(p)[7:-4]
        d = load(p)
        if "kernel" in d:
            rows.append((tag, d))
    print("| config / kernel | CTAs | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    for tag, d in rows:
        cells = []
        for key, _, scale in KEYS:
            v = d.get(key)
            if v is None:
                cells.append("-")
            elif scale is None:
                cells.append(f"{v / d['grid']:,.0f}")
            else:
                cells.append(f"{v * scale:,.1f}")
        print(f"| {tag}: `{d['kernel']}` | {d['grid']:,} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(*sys.argv[1:])
