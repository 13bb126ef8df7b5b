"""Summarise an ncu --set full report: key throughput metrics, stall reasons and a per-region
breakdown of the SASS stall samples.  Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, chunk=50):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__occupancy_limit_registers",
            "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    for k in keys:
        print(f"{k:70s} {d.get(k)} {u.get(k, '')}")
    stalls = []
    for k in hdr:
        m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio$", k)
        if m:
            try:
                stalls.append((float(d[k]), m.group(1)))
            except ValueError:
                pass
    print("stalls per issued instruction:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:8]))
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    h = src[1]
    isrc, iss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in src[2:]:  # the first kernel of the report (a second one starts with its own header)
        if len(r) <= iss or not r[iss].strip().isdigit():
            break
        data.append(r)
    tot = sum(int(r[iss]) for r in data) or 1
    for i in range(0, len(data), chunk):
        part = data[i:i + chunk]
        smp = sum(int(r[iss]) for r in part)
        c = Counter(r[isrc].split()[0] for r in part if r[isrc].split())
        print(f"{i:5d}-{i + len(part) - 1:5d} {100 * smp / tot:5.1f}%  " + " ".join(f"{k}:{v}" for k, v in c.most_common(5)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 50)
