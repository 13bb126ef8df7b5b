exec > gpurun_out/n9.log 2>&1
for s in 6 8 12; do
  ADERSTP_PASS_SLOTS=$s timeout 120 python bench.py --config n9 --steps 10 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slots=$s n9', d['value'], d['roofline']['frac'])"
done
