"""Top stalled SASS instructions of an ncu report with their per-reason stall samples.
Usage: python tools/ncu_hot.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
iss = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_")]
tot = sum(int(r[iss]) for r in data) or 1
agg = {}
for i in stall_cols:
    agg[h[i]] = sum(int(r[i] or 0) for r in data)
print("total samples", tot, "|", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
order = sorted(range(len(data)), key=lambda j: -int(data[j][iss]))
for j in order[:top]:
    r = data[j]
    st = sorted(((int(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{j:5d} {100 * int(r[iss]) / tot:5.2f}%  {r[1][:60]:60s} " + " ".join(f"{n}:{v}" for v, n in st if v))
