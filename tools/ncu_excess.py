"""Shared-memory wavefronts per SASS instruction from an ncu --set full report: the instructions
with the most excessive (bank-conflict) wavefronts, and totals.
Usage: python tools/ncu_excess.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}

    def num(r, k):
        try:
            return float(r[ix[k]].replace(",", ""))
        except (ValueError, KeyError, IndexError):
            return 0.0
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(num(r, "L1 Wavefronts Shared") for r in data)
    exc = sum(num(r, "L1 Wavefronts Shared Excessive") for r in data)
    print(f"shared wavefronts {tot:.4g}, excessive {exc:.4g} ({100 * exc / max(tot, 1):.1f} %)")
    data.sort(key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))
    for r in data[:top]:
        print(f"{r[ix['Address']][-5:]} {num(r, 'L1 Wavefronts Shared Excessive'):12.4g} "
              f"{num(r, 'L1 Wavefronts Shared'):12.4g} {num(r, 'L1 Wavefronts Shared Ideal'):12.4g}  {r[ix['Source']].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
