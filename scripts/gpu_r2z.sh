OUT=gpurun_out/r2z; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:sched_kernel --launch-skip 1 --launch-count 1 --csv \
  --log-file $OUT/dram_default.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu_dram.log 2>&1
echo "dram exit $?"; grep -E "dram__|gpu__time|lts__" $OUT/dram_default.csv | cut -d, -f13-
