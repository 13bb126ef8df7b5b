exec > gpurun_out/corr.log 2>&1
timeout 600 python -m pytest tests/test_gpu_corrector.py -q -x 2>&1 | tail -15
