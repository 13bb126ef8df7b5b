exec > gpurun_out/ts.log 2>&1
python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench
import paper_2003_12787_b200 as S
for n, e in ((8, 50), (8, 50), (4, 80)):
    d = bench.measure_timestep(S, n, e, 10, 3)
    print(n, e, {k: d[k] for k in ('predictor_ms', 'corrector_ms', 'ms_per_step', 'run_simulation_ms_per_step', 'run_simulation_steps', 'run_simulation_stable')})
PY
