# Default bench line (with CPU baseline), its ncu launch list, and the DRAM
# bytes of the policy-run sched_kernel at the same config (roofline.traffic).
#   bash scripts/gpu_bench_default.sh LABEL
OUT=gpurun_out/$1; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench exit $?"; tail -c 2500 $OUT/bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "ref exit $?"; tail -c 1500 $OUT/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > $OUT/launches_bench.log 2>&1
echo "launches exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:sched_kernel --launch-skip 1 --launch-count 1 --csv \
  --log-file $OUT/dram_default.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > $OUT/ncu_dram.log 2>&1
echo "dram exit $?"; grep -E "dram__|gpu__time|lts__" $OUT/dram_default.csv | cut -d, -f13-
