# quick GPU check: the GPU test suite, then one bench line per config given (value, roofline frac)
# usage: bash tools/gpu_quick.sh c2 c3 ...
exec > gpurun_out/quick.log 2>&1
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for cfg in "$@"; do
  v=$(python bench.py --config $cfg --steps 20 --no-e2e --no-cpu-baseline --no-other-configs --no-scaling | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.4g %.4f' % (d['value'], d['roofline']['frac']))")
  echo "$cfg $v"
done
