"""Per-phase clock64 breakdown of the line-pass kernel (experimental build, -DADERSTP_EXPT_TIMING)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ADERSTP_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libaderstp_expt.so")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_12787_b200 as S  # noqa: E402

L = S.lib
L.aderstp_dbg_clock_copy.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.aderstp_dbg_clock2_copy.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.aderstp_dbg_clock3_copy.argtypes = [ctypes.c_void_p, ctypes.c_int]
for cfg_name, elems in (("c3", 32768),):
    cfg = bench.CONFIGS[cfg_name]
    n = cfg["n"]
    q, par = S.generate(cfg["dist"], 1, n, 0, elems, grid=32, layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"])
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"], out_stride=9,
                  par_kind=S.PAR_RHO_CP_CS)
    out = plan.alloc_output(elems)
    for _ in range(3):
        plan.predict(q, 1e-3, par=par, out=out)
    torch.cuda.synchronize()
    host = np.zeros(4096 * 8, dtype=np.int64)
    L.aderstp_dbg_clock3_copy(host.ctypes.data, 4096 * 8)
    t = host.reshape(4096, 8)[:, :5].astype(np.float64)
    d = np.diff(t, axis=1)
    print("dmma8", cfg_name, "per-CTA clocks: staging %.0f  CK %.0f  epilogue(q/favg/face-mma) %.0f  copy-out %.0f" % tuple(np.median(d, axis=0)), "total %.0f" % np.median(t[:, 4] - t[:, 0]))
for cfg_name, elems in (("c2", 32768),):
    cfg = bench.CONFIGS[cfg_name]
    n = cfg["n"]
    q, par = S.generate(cfg["dist"], 1, n, 0, elems, grid=32, layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"])
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"], out_stride=9,
                  par_kind=S.PAR_RHO_CP_CS)
    out = plan.alloc_output(elems)
    for _ in range(3):
        plan.predict(q, 1e-3, par=par, out=out)
    torch.cuda.synchronize()
    host = np.zeros(4096 * 8, dtype=np.int64)
    L.aderstp_dbg_clock2_copy(host.ctypes.data, 4096 * 8)
    t = host.reshape(4096, 8)[:, :6].astype(np.float64)
    d = np.diff(t, axis=1)
    print("dmmap", cfg_name, "per-CTA clocks: staging %.0f  CK %.0f  qavg/favg %.0f  faces %.0f  copy-out %.0f" % tuple(np.median(d, axis=0)), "total %.0f" % np.median(t[:, 5] - t[:, 0]))
for cfg_name, elems in (("c4", 65536), ("n9", 65536)):
    cfg = bench.CONFIGS[cfg_name]
    n = cfg["n"]
    q, par = S.generate(cfg["dist"], 1, n, 0, elems, grid=32, layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"])
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"], out_stride=9,
                  par_kind=S.PAR_RHO_CP_CS)
    out = plan.alloc_output(elems)
    for _ in range(3):
        plan.predict(q, 1e-3, par=par, out=out)
    torch.cuda.synchronize()
    host = np.zeros(4096 * 8, dtype=np.int64)
    L.aderstp_dbg_clock_copy(host.ctypes.data, 4096 * 8)
    t = host.reshape(4096, 8)[:, :5].astype(np.float64)
    d = np.diff(t, axis=1)
    tot = t[:, 4] - t[:, 0]
    print("bip", cfg_name, "per-CTA clocks: staging+TMEM %.0f  CK loop %.0f  qavg/favg %.0f  faces %.0f  total %.0f" % tuple(
        list(np.median(d, axis=0)) + [np.median(tot)]))
