set -e
OUT=gpurun_out/p4; mkdir -p $OUT
python tools/expt_timing.py > $OUT/expt.log 2>&1
python tools/profile_stp.py --config c4 --elems 8192 > $OUT/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stp_bip -s 2 -c 1 -o $OUT/full_c4b python tools/profile_stp.py --config c4 --elems 8192 > $OUT/ncu.log 2>&1
