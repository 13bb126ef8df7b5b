exec > gpurun_out/c4var.log 2>&1
for s in 6 8 12; do
  for c in c4 c3; do
  ADERSTP_NO_DMMA8=1 ADERSTP_PASS_SLOTS=$s python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slots=$s $c', d['value'], d['roofline']['frac'])"
  done
done
