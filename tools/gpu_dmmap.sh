exec > gpurun_out/dmmap.log 2>&1
for lib in tools/libaderstp_old.so paper_2003_12787_b200/libaderstp.so; do
ADERSTP_LIB=$PWD/$lib python - <<'PY'
import sys, json, os
sys.path.insert(0, '.')
import bench, paper_2003_12787_b200 as S
print(os.environ['ADERSTP_LIB'].split('/')[-1])
for name in ('c1', 'c2'):
    cfg = bench.CONFIGS[name]
    r = bench.measure_device(S, cfg, 1, 0, 20, 3, want_clocks=False)
    print(name, cfg['elems'] / (r['ms'] * 1e-3), r['ms'])
for n in (4, 5, 7):
    cfg = dict(n=n, elems=65536, dist=0, q_stride=9)
    r = bench.measure_device(S, cfg, 1, 0, 10, 3, want_clocks=False)
    print('n', n, 65536 / (r['ms'] * 1e-3))
PY
done
