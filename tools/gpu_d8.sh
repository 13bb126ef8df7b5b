exec > gpurun_out/d8.log 2>&1
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for p in 1 0; do
  ADERSTP_DMMA8_PERSIST=$p timeout 120 python bench.py --config c3 --steps 20 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('persist=$p c3', d['value'], d['roofline']['frac'])"
done
