"""Instruction / stall-sample histogram of an ncu report in windows of W SASS lines, with each
window's dominant opcodes.  Usage: python tools/ncu_blocks.py report.ncu-rep elements [W]"""
import collections
import csv
import io
import subprocess
import sys

rep, elems = sys.argv[1], float(sys.argv[2])
W = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, d = rows[1], rows[2:]
ie, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
iw = h.index("L1 Wavefronts Shared")
num = lambda r, i: float(r[i].replace(",", "") or 0)  # noqa: E731
tot_i = sum(num(r, ie) for r in d) / elems
tot_w = sum(num(r, iw) for r in d) / elems
tot_s = sum(num(r, iss) for r in d)
print(f"warp instructions per element {tot_i:.0f}, shared wavefronts per element {tot_w:.0f}, samples {tot_s:.0f}")
for a in range(0, len(d), W):
    blk = d[a:a + W]
    c = collections.Counter()
    for r in blk:
        op = r[1].split()
        if op:
            c[(op[1] if op[0].startswith("@") else op[0]).split(".")[0]] += num(r, ie) / elems
    n = sum(num(r, ie) for r in blk) / elems
    if n == 0:
        continue
    s = sum(num(r, iss) for r in blk)
    wf = sum(num(r, iw) for r in blk) / elems
    print(f"{a:5d} instr {n:7.0f} wf {wf:6.0f} samples {100 * s / tot_s:5.1f}% ",
          " ".join(f"{k}:{v:.0f}" for k, v in c.most_common(6)))
