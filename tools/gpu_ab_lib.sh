# A/B of variant libraries: bash tools/gpu_ab_lib.sh "cfg1 cfg2" lib1 lib2 ...  (lib "" = the product library)
exec >> gpurun_out/ab_lib.log 2>&1
cfgs=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  for cfg in $cfgs; do
    if [ "$lib" = "default" ]; then unset ADERSTP_LIB; else export ADERSTP_LIB=$PWD/tools/libaderstp_$lib.so; fi
    v=$(python bench.py --config $cfg --steps 20 --no-e2e --no-cpu-baseline --no-other-configs --no-scaling | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.4g %.4f' % (d['value'], d['roofline']['frac']))")
    echo "rep$rep lib=$lib cfg=$cfg $v"
  done
done
done
