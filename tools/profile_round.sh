#!/bin/bash
# Produce the round's profiling evidence on a GPU box (run under gpurun from the repo root):
#   1. plain bench run (must exit 0) then the ncu launch list of the same command
#   2. one ncu --set full capture per kernel family (C3 dmma8, C2 dmmap, C4 + nDof 9 bipartite)
set -e
OUT=gpurun_out/prof_${1:-r01}
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $OUT/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1 || true
for cfg in c3 c2 c4 n9; do
  case $cfg in c3) K=stp_dmma8; E=16384;; c2) K=stp_dmmap; E=32768;; c4) K=stp_bip; E=8192;; n9) K=stp_bip; E=8192;; esac
  python tools/profile_stp.py --config $cfg --elems $E > $OUT/plain_$cfg.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $OUT/full_$cfg \
      python tools/profile_stp.py --config $cfg --elems $E > $OUT/ncu_$cfg.log 2>&1 || true
done
python tools/profile_corrector.py > $OUT/plain_corr.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"correct_kernel|surface_kernel" -c 2 -o $OUT/full_corr \
    python tools/profile_corrector.py > $OUT/ncu_corr.log 2>&1 || true
ls -la $OUT
