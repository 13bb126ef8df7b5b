# GPU check used during development: the full -m gpu suite, then the device throughput of the
# main configs (no e2e / CPU baseline), one summary line each
exec > gpurun_out/check.log 2>&1
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
for c in ${CONFIGS:-c3 c2 c4 n9 c1}; do
  python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'], d['ms_per_step'], d['config'].get('cuda_graph'))"
done
