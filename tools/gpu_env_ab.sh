# A/B device throughput of environment settings of the same build:
#   ENVS="X=0 X=1" CONFIGS="c3" bash tools/gpu_env_ab.sh
exec > gpurun_out/envab.log 2>&1
for rep in 1 2; do
for ev in ${ENVS:-NONE=0}; do
for c in ${CONFIGS:-c3}; do
  env $ev python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$ev', '$c', d['value'], d['roofline']['frac'])"
done; done; done
