# Light ncu capture (no source counters) of the policy-run sched_kernel plus
# a DRAM-bytes pass of the bench default:  bash scripts/gpu_ncu_sections.sh LABEL REPLICAS
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 1200 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy \
  --section WarpStateStats --section LaunchStats --section SchedulerStats --clock-control none \
  -k regex:sched_kernel --launch-skip 1 --launch-count 1 -o $OUT/sect -f \
  python bench.py --replicas $2 --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu_sect.log 2>&1
echo "sections exit $?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_sample_count --clock-control none \
  -k regex:sched_kernel --csv --log-file $OUT/dram_default.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu_dram.log 2>&1
echo "dram exit $?"; cat $OUT/dram_default.csv | tail -14
