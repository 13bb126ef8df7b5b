"""Per-step times of the GPU time loop (DESIGN.md section 4.7 table): bench.measure_timestep for
nDof 4 / 8 / 9 / 10 on 80^3 / 50^3 / 44^3 / 40^3 periodic meshes with per-element material."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_12787_b200 as S  # noqa: E402

torch.cuda.set_device(0)
for n, e in ((4, 80), (8, 50), (9, 44), (10, 40)):
    r = bench.measure_timestep(S, n, e, 5, 3)
    print(json.dumps({"n_dof": n, "mesh": e, "predictor_ms": r["predictor_ms"], "corrector_ms": r["corrector_ms"],
                      "run_simulation_ms_per_step": r["run_simulation_ms_per_step"],
                      "run_simulation_elements_per_s": r["run_simulation_elements_per_s"]}), flush=True)
