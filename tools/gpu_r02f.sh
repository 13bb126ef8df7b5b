exec > gpurun_out/r02f.log 2>&1
python -m pytest tests/test_gpu_general.py -q -x 2>&1 | tail -3
python - <<'PY'
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, paper_2003_12787_b200 as S
import torch; torch.cuda.set_device(0)
for m, n in ((21, 8), (21, 4), (12, 6), (9, 8)):
    print(m, n, bench.measure_general_pde(S, 5, 3, m=m, n=n, E=8192 if n >= 8 else 32768))
PY
python tools/table_vs_general.py | grep -v "^{"
