# round-2 first box call: fp64 peaks with clocks, the default bench, the reference arm
exec > gpurun_out/r02a.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python tools/fp64_peaks.py r02 2000
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.json; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r02a_ref.json; echo "ref rc=$?"
