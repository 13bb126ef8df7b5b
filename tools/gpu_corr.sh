timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/corr.log 2>&1
for c in c4 n9 c3; do
python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'])" >> gpurun_out/corr.log
done
python - >> gpurun_out/corr.log 2>&1 <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench
import paper_2003_12787_b200 as S
for n, e in ((8, 50), (4, 80), (10, 40), (9, 44)):
    d = bench.measure_timestep(S, n, e, 10, 3)
    print(n, e, {k: round(d[k], 2) if isinstance(d[k], float) else d[k] for k in ('predictor_ms', 'corrector_ms', 'ms_per_step', 'run_simulation_ms_per_step', 'run_simulation_steps', 'run_simulation_stable')})
PY
