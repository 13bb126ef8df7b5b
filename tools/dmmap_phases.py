"""Per-phase clock64 breakdown of stp_dmmap per CTA for nDof 4..7 (experimental build: make -C
paper_2003_12787_b200 expt): staging, CK loop, qavg/favg, faces, copy-out.
Usage: python tools/dmmap_phases.py [n ...]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ADERSTP_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libaderstp_expt.so")
import torch  # noqa: E402

import paper_2003_12787_b200 as S  # noqa: E402

L = S.lib
L.aderstp_dbg_clock2_copy.argtypes = [ctypes.c_void_p, ctypes.c_int]
for n in [int(x) for x in sys.argv[1:]] or [5, 6, 7]:
    E = 32768
    q, par = S.generate(0, 1, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=9, out_stride=9, par_kind=S.PAR_RHO_CP_CS)
    out = plan.alloc_output(E)
    for _ in range(4):
        plan.predict(q, 1e-3, par=par, out=out)
    torch.cuda.synchronize()
    host = np.zeros(4096 * 8, dtype=np.int64)
    L.aderstp_dbg_clock2_copy(host.ctypes.data, 4096 * 8)
    t = host.reshape(4096, 8)[:, :6].astype(np.float64)
    d = np.diff(t, axis=1)
    print(f"nDof {n} per-CTA clocks: staging %.0f  CK %.0f  qavg/favg %.0f  faces %.0f  copy-out %.0f" % tuple(np.median(d, axis=0)),
          "total %.0f" % np.median(t[:, 5] - t[:, 0]), flush=True)
