exec > gpurun_out/r02e.log 2>&1
python tools/table_vs_general.py
ADERSTP_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --config c3 --e2e-steps 1 --no-other-configs > gpurun_out/bench_gpus2_gloo.json 2> gpurun_out/bench_gpus2_gloo.err
echo "gloo 2-rank rc=$?"
