# round 2: new config parity tests + the DMMA-vs-DFMA A/B timings at C2/C3
exec > gpurun_out/r02c.log 2>&1
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -k "configs or generator or table_pdes or c5 or full_size" -q 2>&1 | tail -15
for env in "" "ADERSTP_NO_DMMAP=1" "ADERSTP_NO_DMMAP=1 ADERSTP_PASS_SLOTS=12" "ADERSTP_NO_DMMAP=1 ADERSTP_PASS_SLOTS=6"; do
  for cfg in c2 c1; do
    echo "== $cfg $env"; env $env python bench.py --config $cfg --steps 20 --no-e2e --no-cpu-baseline --no-other-configs --no-scaling | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
  done
done
for env in "" "ADERSTP_NO_DMMA8=1" "ADERSTP_NO_DMMA8=1 ADERSTP_PASS_SLOTS=12" "ADERSTP_NO_DMMA8=1 ADERSTP_NO_DMMAP=1" "ADERSTP_NO_DMMA8=1 ADERSTP_NO_DMMAP=1 ADERSTP_PASS_SLOTS=12"; do
  echo "== c3 $env"; env $env python bench.py --config c3 --steps 20 --no-e2e --no-cpu-baseline --no-other-configs --no-scaling | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
done
# ncu A/B (one launch each): DMMA kernels vs the DFMA line-pass kernel, C2 and C3
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__instruction_throughput.avg.pct_of_peak_sustained_active,sm__inst_issued.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum
for spec in "c2::" "c2:ADERSTP_NO_DMMAP=1:" "c3::" "c3:ADERSTP_NO_DMMA8=1:"; do
  cfg=${spec%%:*}; rest=${spec#*:}; env=${rest%%:*}
  tag=$cfg$( [ -n "$env" ] && echo _dfma || echo _dmma )
  env $env ncu --metrics $M --clock-control none -k regex:stp_ -s 3 -c 1 --csv python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-other-configs --no-scaling > gpurun_out/ncu_ab_$tag.csv 2>&1
  echo "ncu $tag rc=$?"
done
