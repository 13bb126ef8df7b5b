# A/B device throughput of several library builds (ADERSTP_LIB) on the same box:
#   LIBS="tools/libaderstp_old.so paper_2003_12787_b200/libaderstp.so" CONFIGS="c3" bash tools/gpu_ab.sh
exec > gpurun_out/ab.log 2>&1
LIBS=${LIBS:-"tools/libaderstp_old.so paper_2003_12787_b200/libaderstp.so"}
for rep in 1 2; do
for lib in $LIBS; do
for c in ${CONFIGS:-c3}; do
  ADERSTP_LIB=$PWD/$lib python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], '$c', d['value'], d['roofline']['frac'])"
done; done; done
