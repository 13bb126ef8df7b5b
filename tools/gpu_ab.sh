# A/B of an environment switch on the same box
exec > gpurun_out/ab.log 2>&1
for rep in 1 2; do for v in 0 1; do for c in ${CONFIGS:-c2}; do
  if [ $v = 1 ]; then export ADERSTP_COOP_FACES=1; else unset ADERSTP_COOP_FACES; fi
  python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v=$v $c', d['value'], d['roofline']['frac'])"
done; done; done
