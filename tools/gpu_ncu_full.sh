# ncu --set full (one launch) of the STP kernel of each config given: bash tools/gpu_ncu_full.sh tag cfg...
tag=$1; shift
for cfg in "$@"; do
  ncu --set full --import-source on --clock-control none -k regex:stp_ -s 3 -c 1 \
      -o gpurun_out/ncu_${tag}_${cfg} python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e \
      --no-cpu-baseline --no-other-configs --no-scaling > gpurun_out/ncu_${tag}_${cfg}.log 2>&1
  echo "$cfg rc=$?" >> gpurun_out/ncu_${tag}.status
done
