#!/usr/bin/env python3
"""Parity and timing of the warp-per-element kernel (ADERSTP_WPE=1) against the oracle and the
padded-DMMA kernel at nDof 4 / 6."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2003_12787_b200 as S  # noqa: E402

orc = O.Oracle()


def run(n, E, wpe, qs=9):
    os.environ["ADERSTP_WPE"] = "1" if wpe else "0"
    q, par = S.generate(0, 42 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=qs)
    par_h = par.cpu().numpy()
    dt = O.cfl_dt(n, float(par_h[:, 1].max()))
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=qs, par_kind=S.PAR_RHO_CP_CS)
    out = plan.predict(q, dt, par=par)
    plan.status()
    torch.cuda.synchronize()
    ref = orc.stp(n, 9, orc.from_aosoa(n, 9, qs, q.cpu().numpy()), dt, par=orc.material_lmr(par_h))
    got = orc.from_aosoa(n, 9, 9, out.qavg.cpu().numpy())
    errs = [O.per_element_rel_diff(ref.qavg, got),
            O.per_element_rel_diff(ref.face_q.reshape(E, -1), out.face_q.cpu().numpy().reshape(E, -1)),
            O.per_element_rel_diff(ref.face_f.reshape(E, -1), out.face_f.cpu().numpy().reshape(E, -1))]
    fa = np.stack([orc.from_aosoa(n, 9, 9, out.favg[:, d].cpu().numpy()) for d in range(3)], 1)
    errs.append(O.per_element_rel_diff(ref.favg.reshape(E, -1), fa.reshape(E, -1)))
    return errs


def timeit(n, E, wpe, reps=20):
    os.environ["ADERSTP_WPE"] = "1" if wpe else "0"
    q, par = S.generate(0, 7, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    dt = O.cfl_dt(n, 6.0)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    out = plan.predict(q, dt, par=par)
    for _ in range(3):
        plan.predict(q, dt, par=par, out=out)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        plan.predict(q, dt, par=par, out=out)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / reps
    return E / ms * 1e3


if __name__ == "__main__":
    for n in (6, 5, 4):
        for E, qs in ((1, 9), (50, 9), (1037, 9), (50, 12)):
            try:
                e = run(n, E, True, qs)
                print(f"wpe n={n} E={E} qs={qs} errs qavg/face_q/face_f/favg = " + " ".join(f"{x:.2e}" for x in e), flush=True)
            except Exception as ex:  # noqa: BLE001
                print(f"wpe n={n} E={E} qs={qs} FAILED: {ex}", flush=True)
    for n, E in ((6, 32768), (5, 65536), (4, 131072)):
        for wpe in (False, True):
            print(f"n={n} E={E} wpe={wpe}: {timeit(n, E, wpe) / 1e6:.2f} M elem/s", flush=True)
