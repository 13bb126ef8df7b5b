"""Driver for ncu captures of the corrector kernels: a 50^3 nDof-8 mesh, one predictor launch
(1/h-scaled material), then the full corrector (qavg staged, volume + surface) and one fused
run_simulation step (the predictor applies the volume term; surface-only corrector).
ncu -k regex:correct_kernel -c 2 selects the two corrector launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2003_12787_b200 as S  # noqa: E402

n, e = 8, 50
E = e ** 3
q, par = S.generate(0, 7, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
rho, cp, cs = par[:, 0], par[:, 1], par[:, 2]
mu = rho * cs * cs
lam = rho * cp * cp - 2.0 * mu
s = float(e)
par_s = torch.stack([lam * s, mu * s, rho / s], 1).contiguous()
pred = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_LAMBDA_MU_RHO)
corr = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
out = pred.alloc_output(E, want_favg=False)
dt = 0.35 / e / (3.0 * float(cp.max()) * (2 * n - 1))
pred.predict(q, dt, par=par_s, out=out, want_favg=False)
corr.correct(q, e, out, par=par)
corr.run_simulation(q, e, dt, par=par, cfl=0.35)
torch.cuda.synchronize()
corr.status()
print("ok corrector", E)
