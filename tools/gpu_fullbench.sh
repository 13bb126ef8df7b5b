# full default bench (driver contract), the reference arm, and the C5 strong-scaling config at N=1
exec > gpurun_out/fullbench.log 2>&1
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rc=$?
python bench.py --config c5 --no-other-configs > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$?
