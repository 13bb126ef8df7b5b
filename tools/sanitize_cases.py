#!/usr/bin/env python3
"""One small invocation of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Run as:  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
Each case is checked against the CPU oracle (so a sanitizer run is also a parity run)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2003_12787_b200 as S  # noqa: E402

orc = O.Oracle()
E = int(os.environ.get("SANITIZE_ELEMS", "3"))


def elastic(n, env=None, layout=S.LAYOUT_AOSOA, qs=9):
    for k in ("ADERSTP_NO_DMMA8", "ADERSTP_NO_DMMAP", "ADERSTP_PASS_SLOTS", "ADERSTP_FORCE_GENERIC"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    q, par = S.generate(0, 7 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    dt = O.cfl_dt(n, float(par[:, 1].max()))
    ref = orc.stp(n, 9, orc.from_aosoa(n, 9, 9, q.cpu().numpy()), dt, par=orc.material_lmr(par.cpu().numpy()))
    if layout == S.LAYOUT_AOS:
        qa = torch.empty(E, n ** 3 * 16, dtype=torch.float64, device="cuda")
        S.convert_layout(n, 9, E, S.LAYOUT_AOSOA, 9, q, S.LAYOUT_AOS, 16, qa)
        plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOS, q_stride=16, out_stride=16, par_kind=S.PAR_RHO_CP_CS)
        out = plan.predict(qa, dt, par=par)
        got = out.qavg.cpu().numpy().reshape(E, n ** 3, 16)[:, :, :9].reshape(E, -1)
    else:
        plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
        out = plan.predict(q, dt, par=par)
        got = orc.from_aosoa(n, 9, 9, out.qavg.cpu().numpy())
    plan.status()
    err = max(O.per_element_rel_diff(ref.qavg, got),
              O.per_element_rel_diff(ref.face_f.reshape(E, -1), out.face_f.cpu().numpy().reshape(E, -1)))
    return err


def table(n, m=3):
    rng = np.random.default_rng(n)
    qn = rng.uniform(-1, 1, (E, n ** 3 * m))
    plan = S.Plan(n, S.advection_pde((1.0, 0.5, 0.25), m), layout=S.LAYOUT_AOSOA, q_stride=m, out_stride=m)
    out = plan.predict(torch.from_numpy(orc.to_aosoa(n, m, m, qn)).cuda(), 2e-3)
    plan.status()
    ref = orc.stp(n, m, qn, 2e-3, pde_kind=O.PDE_ADVECTION, args=[1.0, 0.5, 0.25])
    return O.per_element_rel_diff(ref.qavg, orc.from_aosoa(n, m, m, out.qavg.cpu().numpy()))


def timeloop(n, e=2):
    rng = np.random.default_rng(3)
    u0 = rng.standard_normal((e ** 3, n ** 3 * 9))
    plan = S.Plan(n, S.elastic_pde(2.0, 1.0, 1.0), layout=S.LAYOUT_AOSOA)
    u = torch.from_numpy(orc.to_aosoa(n, 9, 9, u0)).cuda()
    t_end = 2 * 0.35 * (1.0 / e) / (3.0 * 2.0 * (2 * n - 1))
    ok, steps, _ = plan.run_simulation(u, e, t_end, cfl=0.35)
    torch.cuda.synchronize()
    return 0.0 if ok and steps == 2 else 1.0


CASES = [
    ("stp_dmma8 nDof 8", lambda: elastic(8)),
    ("stp_dmma8<AOS> nDof 8", lambda: elastic(8, layout=S.LAYOUT_AOS)),
    ("stp_dmmap nDof 4", lambda: elastic(4)),
    ("stp_dmmap nDof 6", lambda: elastic(6)),
    ("stp_dmmap<AOS> nDof 6", lambda: elastic(6, layout=S.LAYOUT_AOS)),
    ("stp_bip nDof 9", lambda: elastic(9)),
    ("stp_bip nDof 10", lambda: elastic(10)),
    ("stp_bip<AOS> nDof 10", lambda: elastic(10, layout=S.LAYOUT_AOS)),
    ("stp_pass nDof 3", lambda: elastic(3)),
    ("stp_pass nDof 8 (NO_DMMA8)", lambda: elastic(8, {"ADERSTP_NO_DMMA8": "1"})),
    ("stp_kernel generic nDof 5", lambda: elastic(5, {"ADERSTP_FORCE_GENERIC": "1"})),
    ("aos staged transposes nDof 3", lambda: elastic(3, layout=S.LAYOUT_AOS)),
    ("stp_dmma8_table nDof 8", lambda: table(8)),
    ("stp_kernel table nDof 5", lambda: table(5)),
    ("time loop nDof 8 (fused dmma8 + surface)", lambda: timeloop(8)),
    ("time loop nDof 6 (fused dmmap + surface)", lambda: timeloop(6)),
    ("time loop nDof 10 (fused bip + surface)", lambda: timeloop(10)),
]

if __name__ == "__main__":
    only = sys.argv[1:]
    worst = 0.0
    for name, fn in CASES:
        if only and not any(o in name for o in only):
            continue
        err = fn()
        worst = max(worst, err)
        print(f"{name}: worst rel_diff {err:.3e}", flush=True)
    torch.cuda.synchronize()
    assert worst <= 1e-11, worst
    print("sanitize cases done")
