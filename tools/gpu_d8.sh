exec > gpurun_out/d8.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
for i in 1 2; do
python bench.py --config c3 --steps 20 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['roofline']['frac'])"
done
