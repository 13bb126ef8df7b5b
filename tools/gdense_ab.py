"""Dense user LinearPde at nDof 8: stp_gdense (DMMA GEMMs) against the scalar general kernel
(ADERSTP_NO_GDENSE=1), M elem/s per m, device-resident.  Usage: python tools/gdense_ab.py [m ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2003_12787_b200 as S  # noqa: E402

ms = [int(x) for x in sys.argv[1:]] or [6, 9, 12, 16, 21]
for m in ms:
    row = []
    for flag in ("0", "1"):
        os.environ["ADERSTP_NO_GDENSE"] = flag
        E = 16384 if flag == "0" else 4096
        r = bench.measure_general_pde(S, 5, 3, m=m, n=8, E=E)
        row.append(r["elements_per_s"] / 1e6)
    print(f"m={m:2d}  gdense {row[0]:8.3f} M elem/s   general {row[1]:8.3f} M elem/s   x{row[0] / row[1]:.2f}", flush=True)
