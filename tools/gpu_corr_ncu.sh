# ncu durations / DRAM bytes of the two corrector kernels (full, surface-only) of tools/profile_corrector.py
exec > gpurun_out/corr_ncu.log 2>&1
for lib in ${LIBS:-tools/libaderstp_old.so paper_2003_12787_b200/libaderstp.so}; do
  echo "== $lib"
  ADERSTP_LIB=$PWD/$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"correct_kernel|surface_kernel" -c 2 --csv python tools/profile_corrector.py 2>/dev/null | grep -E "correct_kernel|surface_kernel" | \
    awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}'
done
