# quick GPU check: parity tests + device throughput per config (no e2e / cpu baseline)
exec > gpurun_out/quick.log 2>&1
python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in ${CONFIGS:-c3}; do
  python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'], d['clocks'])"
done
[ -n "$EXPT" ] && python tools/expt_timing.py
