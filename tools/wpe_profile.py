#!/usr/bin/env python3
"""A few launches of the warp-per-element kernel for ncu:
ncu --set full --import-source on --clock-control none -k regex:stp_wpe -s 3 -c 1 -o out python tools/wpe_profile.py 4 131072"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ADERSTP_WPE"] = "1"
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2003_12787_b200 as S  # noqa: E402

n, E = int(sys.argv[1]), int(sys.argv[2])
q, par = S.generate(0, 7, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
dt = O.cfl_dt(n, 6.0)
out = plan.predict(q, dt, par=par)
for _ in range(5):
    plan.predict(q, dt, par=par, out=out)
torch.cuda.synchronize()
