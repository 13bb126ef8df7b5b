#!/usr/bin/env python3
"""Table PDEs (the reference's advection / demo / a 4-nonzero probed system) on the term-table
kernels (stp_kernel generic, stp_dmma8_table at nDof 8) vs the general kernel (ADERSTP_GENERAL=1),
elements/s per order: decides the dispatch of user PDEs."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_12787_b200 as S  # noqa: E402


def rate(n, pde, m, E, general):
    os.environ["ADERSTP_GENERAL"] = "1" if general else "0"
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.rand(E, n ** 3 * m, dtype=torch.float64, device="cuda", generator=g) - 0.5
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=m, out_stride=m)
    out = plan.alloc_output(E)
    for _ in range(3):
        plan.predict(q, 1e-3, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.predict(q, 1e-3, out=out)
    e1.record()
    torch.cuda.synchronize()
    plan.status()
    return E / (e0.elapsed_time(e1) / 10 * 1e-3)


rng = np.random.default_rng(5)
A = []
for d in range(3):
    a = np.zeros((9, 9))
    for r in range(9):
        a[r, rng.choice(9, 3, replace=False)] = rng.uniform(-1, 1, 3)
    A.append(a)
cases = {"advection_m8": (S.advection_pde((1.0, 0.5, 0.25), 8), 8), "demo_m6": (S.paper_demo_pde(), 6),
         "probed_m9_3nnz": (S.linear_pde(A), 9)}
res = {}
for name, (pde, m) in cases.items():
    for n in (3, 4, 5, 6, 7, 8, 9, 10):
        E = 16384 if n <= 6 else 8192
        t, g = rate(n, pde, m, E, False), rate(n, pde, m, E, True)
        res[f"{name}_n{n}"] = {"table": t, "general": g, "ratio_general_over_table": g / t}
        print(name, n, f"table {t:.4g}  general {g:.4g}  ratio {g / t:.2f}", flush=True)
print(json.dumps(res))
