# round-2 profiles: ncu --set full of the tuned kernel of c3, c2, c4, n9 and the launch list of the default bench
exec > gpurun_out/r02g.log 2>&1
bash tools/gpu_ncu_full.sh r02 c3 c4 n9 c2
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_r02_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r02_launches.log 2>&1
echo "launches rc=$?"
