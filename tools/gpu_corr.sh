timeout 600 python -m pytest tests/test_gpu_corrector.py -q -x > gpurun_out/corr.log 2>&1
bash tools/gpu_ts.sh
