import ctypes, os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
os.environ["ADERSTP_LIB"] = "/root/repo/tools/libaderstp_expt.so"
import torch, bench
import paper_2003_12787_b200 as S
L = S.lib
for fn in ("aderstp_dbg_clock2_copy", "aderstp_dbg_clock3_copy"):
    getattr(L, fn).argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = bench.CONFIGS["c3"]; n = 8; elems = 32768
q, par = S.generate(0, 1, n, 0, elems, layout=S.LAYOUT_AOSOA, q_stride=12)
for nod in ("0",):
    os.environ["ADERSTP_NO_DMMA8"] = nod
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=12, out_stride=9, par_kind=S.PAR_RHO_CP_CS)
    out = plan.alloc_output(elems)
    for _ in range(3): plan.predict(q, 1e-3, par=par, out=out)
    torch.cuda.synchronize()
    host = np.zeros(4096 * 8, dtype=np.int64)
    if nod == "0":
        L.aderstp_dbg_clock3_copy(host.ctypes.data, 4096 * 8); k = 7
    else:
        L.aderstp_dbg_clock2_copy(host.ctypes.data, 4096 * 8); k = 6
    t = host.reshape(4096, 8)[:, :k].astype(np.float64)
    print("NO_DMMA8", nod, "phases", np.median(np.diff(t, axis=1), axis=0).round(), "total", np.median(t[:, k-1] - t[:, 0]))
