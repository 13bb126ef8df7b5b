"""The BASELINE metric against order: elastic STP elements/s, algorithmic fp64 GFLOP/s and the
fraction of the per-order roofline (min of fp64 peak / FLOP(n), HBM / Byte(n)) for nDof 2..10 on
one B200.  Workload per order: U[-1,1] data, per-element material, compact AoSoA (q stride 9),
elements sized so inputs + outputs exceed the L2 (>= 1 GB per step); device-resident, CUDA events,
the bench's dt.  Prints one JSON line per order and a markdown table.
Usage: python tools/order_sweep.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_12787_b200 as S  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
torch.cuda.set_device(0)
rows = []
for n in range(2, 11):
    byte_e = S.byte_count(n, 9, True)
    E = max(32768, int(2e9 // byte_e) // 1024 * 1024)  # >= 2 GB of traffic per step
    E = min(E, 262144)
    cfg = dict(n=n, elems=E, dist=0, q_stride=9)
    r = bench.measure_device(S, cfg, 1, 0, steps, 3, want_clocks=True)
    v = E / (r["ms"] * 1e-3)
    rf = bench.roofline_of(S, n, v, E, None)
    row = {"n_dof": n, "order": n - 1, "elements": E, "elements_per_s": v, "ms_per_step": r["ms"],
           "fp64_gflops": v * rf["flop_per_element"] / 1e9, "achieved_gbs": v * rf["byte_per_element"] / 1e9,
           "bound": rf["bound"], "frac_of_roofline": rf["frac"], "roofline_elements_per_s": rf["roofline_elements_per_s"],
           "sm_mhz": (r["clocks"] or {}).get("sm_mhz"), "reasons": (r["clocks"] or {}).get("reasons")}
    rows.append(row)
    print(json.dumps(row), flush=True)
print("| nDof (order) | elements | M elem/s | fp64 GFLOP/s | GB/s | bound | % of roofline |")
print("|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r['n_dof']} ({r['order']}) | {r['elements']:,} | {r['elements_per_s'] / 1e6:.2f} | "
          f"{r['fp64_gflops']:,.0f} | {r['achieved_gbs']:,.0f} | {r['bound']} | {100 * r['frac_of_roofline']:.1f} |")
