# corrector tests + time-step measurement for two library builds (ADERSTP_LIB)
exec > gpurun_out/corr.log 2>&1
timeout 600 python -m pytest tests/test_gpu_corrector.py -q -x 2>&1 | tail -2
for lib in ${LIBS:-tools/libaderstp_old.so paper_2003_12787_b200/libaderstp.so}; do
ADERSTP_LIB=$PWD/$lib python - <<'PY'
import os, sys
sys.path.insert(0, '.')
import bench
import paper_2003_12787_b200 as S
for n, e in ((8, 50), (4, 80), (10, 40), (9, 44)):
    d = bench.measure_timestep(S, n, e, 20, 3)
    print(os.path.basename(os.environ["ADERSTP_LIB"]), n, e, {k: round(d[k], 2) if isinstance(d[k], float) else d[k] for k in ('predictor_ms', 'corrector_ms', 'corrector_hbm_frac', 'run_simulation_ms_per_step')})
PY
done
