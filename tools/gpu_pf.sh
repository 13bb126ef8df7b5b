exec > gpurun_out/pf.log 2>&1
for pf in 0 148 296; do for c in c2 c3 c4 n9; do
  ADERSTP_PREFETCH=$pf python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf=$pf $c', d['value'], d['roofline']['frac'])"
done; done
