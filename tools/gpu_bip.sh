exec > gpurun_out/bip.log 2>&1
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for c in n9 c4; do
  timeout 120 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'])"
done
python tools/expt_timing.py 2>&1 | grep bip
