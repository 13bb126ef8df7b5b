"""Throughput of the generic table kernel (user LinearPde path): the elastic system given as
probed flux matrices (ADERSTP_PDE_LINEAR, m = 9) and an advection system, device-resident."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_12787_b200 as S  # noqa: E402


def elastic_A(lam, mu, rho):
    A = [np.zeros((9, 9)) for _ in range(3)]
    L = lam + 2 * mu
    for d in range(3):
        vel = 6 + d
        A[d][d, vel] = L
        for o in range(3):
            if o != d:
                A[d][o, vel] = lam
    A[0][3, 7] = mu; A[0][4, 8] = mu; A[1][3, 6] = mu; A[1][5, 8] = mu; A[2][4, 6] = mu; A[2][5, 7] = mu
    A[0][6, 0] = A[0][7, 3] = A[0][8, 4] = 1 / rho
    A[1][6, 3] = A[1][7, 1] = A[1][8, 5] = 1 / rho
    A[2][6, 4] = A[2][7, 5] = A[2][8, 2] = 1 / rho
    return A


lib = os.path.basename(os.environ.get("ADERSTP_LIB", "libaderstp.so"))
for n, E in ((4, 32768), (6, 16384), (8, 8192), (9, 4096), (10, 4096)):
    pde = S.linear_pde(elastic_A(2.0, 1.0, 1.5))
    q = torch.randn(E, n ** 3 * 9, dtype=torch.float64, device="cuda")
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=9, out_stride=9)
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
    print(lib, "linear-elastic", n, "%.3f M elem/s" % (E / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e6))

for name, pde, m in (("advection-m8", S.advection_pde((1.0, 0.5, 0.25), 8), 8), ("demo-m6", S.paper_demo_pde(), 6)):
    n, E = 8, 16384
    q = torch.randn(E, n ** 3 * m, dtype=torch.float64, device="cuda")
    for generic in ("0", "1"):
        os.environ["ADERSTP_FORCE_GENERIC"] = generic
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
        print(lib, name, n, "generic" if generic == "1" else "default", "%.3f M elem/s" % (E / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e6))
    os.environ["ADERSTP_FORCE_GENERIC"] = "0"
