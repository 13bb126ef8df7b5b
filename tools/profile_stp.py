"""Small driver for ncu captures: generate one config's inputs, run W warm-up launches and one
more launch of the STP kernel (ncu -k regex:stp_kernel -s W -c 1 selects it)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_12787_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--elems", type=int, default=16384)
ap.add_argument("--warmup", type=int, default=2)
a = ap.parse_args()
cfg = dict(bench.CONFIGS[a.config])
cfg["elems"] = a.elems
n = cfg["n"]
grid = round(a.elems ** (1 / 3)) if cfg["dist"] == 2 else 1
q, par = S.generate(cfg["dist"], bench.SEED, n, 0, a.elems, grid=grid, layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"])
dt = S.stable_dt(n, float(par[:, 1].max()), cfl=0.5)
plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"], out_stride=9,
              par_kind=S.PAR_RHO_CP_CS)
out = plan.alloc_output(a.elems)
for _ in range(a.warmup + 1):
    plan.predict(q, dt, par=par, out=out)
torch.cuda.synchronize()
plan.status()
print("ok", a.config, a.elems)
