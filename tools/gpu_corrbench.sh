# corrector tests + the time-step measurement (predictor, full corrector, fused loop)
exec > gpurun_out/corr.log 2>&1
timeout 600 python -m pytest tests/test_gpu_corrector.py -q -x 2>&1 | tail -2
python - <<'PY'
import sys
sys.path.insert(0, '.')
import bench
import paper_2003_12787_b200 as S
for n, e in ((8, 50), (4, 80), (10, 40)):
    d = bench.measure_timestep(S, n, e, 10, 3)
    print(n, e, {k: round(d[k], 2) if isinstance(d[k], float) else d[k] for k in ('predictor_ms', 'corrector_ms', 'run_simulation_ms_per_step', 'corrector_achieved_gbs')})
PY
