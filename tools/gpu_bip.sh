exec > gpurun_out/bip.log 2>&1
python tools/dbg_bip.py 2>&1 | head -3
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
ADERSTP_PASS_SLOTS=12 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for s in 0 12; do for c in c4; do
  ADERSTP_PASS_SLOTS=$s timeout 120 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slots=$s $c', d['value'], d['roofline']['frac'])"
done; done
python tools/expt_timing.py 2>&1 | grep bip
