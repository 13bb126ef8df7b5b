"""Driver for ncu captures of the table-PDE line-pass kernel (stp_tlp): advection m = 8 or the
demo system at nDof 9 / 10, 8,192 elements, 4 launches (ncu -k regex:stp_tlp -s 3 -c 1).
Usage: python tools/tlp_profile.py [n] [advection|demo]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2003_12787_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
kind = sys.argv[2] if len(sys.argv) > 2 else "advection"
pde, m = (S.advection_pde((1.0, 0.5, 0.25), 8), 8) if kind == "advection" else (S.paper_demo_pde(), 6)
E = 8192
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.rand(E, n ** 3 * m, dtype=torch.float64, device="cuda", generator=g) - 0.5
plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=m, out_stride=m)
out = plan.alloc_output(E)
for _ in range(4):
    plan.predict(q, 1e-3, out=out)
torch.cuda.synchronize()
plan.status()
print("ok", n, kind, E)
