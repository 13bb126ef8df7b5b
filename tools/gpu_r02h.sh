exec > gpurun_out/r02h.log 2>&1
python -m pytest tests/test_gpu_general.py tests/test_gpu_corrector.py -q -x 2>&1 | tail -2
python - <<'PY'
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, paper_2003_12787_b200 as S
import torch; torch.cuda.set_device(0)
for m, n in ((21, 8), (21, 4), (12, 6), (9, 8), (21, 10)):
    print(m, n, bench.measure_general_pde(S, 5, 3, m=m, n=n, E=8192 if n >= 8 else 32768)["elements_per_s"])
PY
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"surface|dmma8|scale" --csv --log-file gpurun_out/ncu_corr_r02.csv python - <<'PY'
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, paper_2003_12787_b200 as S, torch
torch.cuda.set_device(0)
print(bench.measure_timestep(S, 8, 50, 2, 3))
PY
