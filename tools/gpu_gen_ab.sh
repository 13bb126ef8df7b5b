exec > gpurun_out/gen_ab.log 2>&1
for lib in default gen512; do
  if [ "$lib" = "default" ]; then unset ADERSTP_LIB; else export ADERSTP_LIB=$PWD/tools/libaderstp_$lib.so; fi
  python - <<'PY'
import os, sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, paper_2003_12787_b200 as S
import torch; torch.cuda.set_device(0)
lib = os.environ.get("ADERSTP_LIB", "default")
for m, n in ((21, 8), (21, 4), (12, 6), (8, 10), (8, 9)):
    print(lib, m, n, bench.measure_general_pde(S, 5, 3, m=m, n=n, E=8192 if n >= 8 else 32768)["elements_per_s"], flush=True)
PY
done
