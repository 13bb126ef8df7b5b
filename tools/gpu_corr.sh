timeout 600 python -m pytest tests/test_gpu_corrector.py -q -x > gpurun_out/corr.log 2>&1
timeout 600 python -m pytest tests -q -x -m gpu >> gpurun_out/corr.log 2>&1
bash tools/gpu_ts.sh
python bench.py --config c3 --steps 20 --no-e2e --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['roofline']['frac'])" >> gpurun_out/corr.log
