"""Shared-memory wavefronts per SASS instruction of an ncu --set full report (source page):
total, ideal and excessive (bank-conflict) wavefronts, the top offenders with their source line.
Usage: python tools/ncu_smem.py report.ncu-rep [top] [elements]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
elems = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h, data = rows[hi], rows[hi + 1:]
ci = {k: h.index(k) for k in ("Address", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                                "L1 Wavefronts Shared Excessive")}
ci["Source"] = len(h) - 1 - h[::-1].index("Source")  # the SASS text
ci["Line"] = h.index("Line No") if "Line No" in h else None
def num(r, k):
    try:
        return float(r[ci[k]].replace(",", ""))
    except ValueError:
        return 0.0
# source-line rows (no address) aggregate the SASS rows below them: keep only the latter
sm, seen = [], set()
for r in data:  # a SASS row is listed under every (inlined) source line it belongs to: dedupe
    if len(r) == len(h) and r[ci["Address"]].startswith("0x") and num(r, "L1 Wavefronts Shared") > 0:
        if r[ci["Address"]] not in seen:
            seen.add(r[ci["Address"]])
            sm.append(r)
line_of = {}
cur = None
for r in data:
    if len(r) == len(h) and not r[ci["Address"]].startswith("0x"):
        cur = r[ci["Line"]] if ci["Line"] is not None else None
    elif len(r) == len(h):
        line_of[id(r)] = cur
tw = sum(num(r, "L1 Wavefronts Shared") for r in sm)
ti = sum(num(r, "L1 Wavefronts Shared Ideal") for r in sm)
te = sum(num(r, "L1 Wavefronts Shared Excessive") for r in sm)
print(f"shared wavefronts {tw / elems:.0f}  ideal {ti / elems:.0f}  excessive {te / elems:.0f}  (per element)")
for r in sorted(sm, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:top]:
    print(f"{r[ci['Address']]:>6} {num(r, 'L1 Wavefronts Shared') / elems:8.1f} ideal {num(r, 'L1 Wavefronts Shared Ideal') / elems:8.1f} "
          f"exc {num(r, 'L1 Wavefronts Shared Excessive') / elems:7.1f}  L{line_of.get(id(r))} {r[ci['Source']][:60]}")
