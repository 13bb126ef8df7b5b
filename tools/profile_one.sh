#!/bin/bash
# One ncu --set full capture of one config's tuned kernel (development): profile_one.sh CFG KERNEL ELEMS TAG
OUT=gpurun_out/one; mkdir -p $OUT
python tools/profile_stp.py --config $1 --elems $3 > $OUT/plain_$4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o $OUT/full_$4 \
    python tools/profile_stp.py --config $1 --elems $3 > $OUT/ncu_$4.log 2>&1
