"""Debug helper: per-field qavg error of the nDof-10 kernel vs the oracle for a few dt."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
import paper_2003_12787_b200 as S
orc = O.Oracle()
n = 10
E = 3
q, par = S.generate(0, 1244, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
par_h = par.cpu().numpy()
qc = orc.from_aosoa(n, 9, 9, q.cpu().numpy())
for dt in (1e-12, 1e-3, O.cfl_dt(n, par_h[:, 1].max())):
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    out = plan.predict(q, dt, par=par)
    plan.status()
    ref = orc.stp(n, 9, qc, dt, par=orc.material_lmr(par_h))
    qa = orc.from_aosoa(n, 9, 9, out.qavg.cpu().numpy()).reshape(E, n, n, n, 9)
    rq = ref.qavg.reshape(E, n, n, n, 9)
    err = np.abs(qa - rq).max(axis=(0, 1, 2, 3)) / (np.abs(rq).max() + 1e-300)
    print("dt", dt, "per-field rel err", np.array2string(err, precision=2))
    if dt == 1e-3:
        d = np.abs(qa - rq)[0, :, :, :, 6]
        idx = np.unravel_index(np.argmax(d), d.shape)
        print("  worst u node (k3,k2,k1)", idx, "gpu", qa[0][idx][6], "ref", rq[0][idx][6])
        print("  u err by k3", np.array2string(d.max(axis=(1, 2)), precision=1))
        print("  u err by k2", np.array2string(d.max(axis=(0, 2)), precision=1))
        print("  u err by k1", np.array2string(d.max(axis=(0, 1)), precision=1))
