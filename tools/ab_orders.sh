# A/B of variant libraries on the elastic STP at the given nDof values (32,768 elements each):
# bash tools/ab_orders.sh "5 7" lib1 lib2 ...  (lib "default" = the product library)
exec >> gpurun_out/ab_orders.log 2>&1
orders=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  if [ "$lib" = "default" ]; then unset ADERSTP_LIB; else export ADERSTP_LIB=$PWD/tools/libaderstp_$lib.so; fi
  for n in $orders; do
    v=$(python -c "
import sys; sys.path.insert(0, '.')
import torch, bench, paper_2003_12787_b200 as S
torch.cuda.set_device(0)
r = bench.measure_device(S, dict(n=$n, elems=32768, dist=0, q_stride=9), 1, 0, 10, 3, want_clocks=False)
print('%.4g' % (32768 / (r['ms'] * 1e-3)))")
    echo "rep$rep lib=$lib nDof=$n $v"
  done
done
done
