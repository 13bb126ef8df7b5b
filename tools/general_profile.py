"""Driver for ncu captures of the general kernel (stp_general): a dense LinearPde (every A_d, B_d
entry nonzero) with m quantities at nDof n, 4 launches (ncu -k regex:stp_general -s 3 -c 1).
Usage: python tools/general_profile.py [m] [n] [elements]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_12787_b200 as S  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 21
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
E = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
rng = np.random.default_rng(7)
A = [rng.uniform(-1, 1, (m, m)) / m for _ in range(3)]
B = [rng.uniform(-0.5, 0.5, (m, m)) / m for _ in range(3)]
pde = S.linear_pde(A, B)
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.rand(E, n ** 3 * m, dtype=torch.float64, device="cuda", generator=g) - 0.5
plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=m, out_stride=m)
out = plan.alloc_output(E)
for _ in range(4):
    plan.predict(q, 1e-3, out=out)
torch.cuda.synchronize()
plan.status()
print("ok", m, n, E)
