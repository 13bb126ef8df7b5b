exec > gpurun_out/ts.log 2>&1
python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench
import paper_2003_12787_b200 as S
for n, e in ((8, 50), (4, 80), (10, 40)):
    print(json.dumps(bench.measure_timestep(S, n, e, 10, 3)))
PY
