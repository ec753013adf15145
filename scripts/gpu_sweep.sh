set -u
OUT=gpurun_out/r1b; mkdir -p $OUT
python scripts/time_case.py c2_pascal 1 > $OUT/time_case.txt 2>&1
python scripts/time_case.py c2_fcfs 1 >> $OUT/time_case.txt 2>&1
for r in 592 888 1184 1480 1776 2072 2368 2960; do
  timeout 300 python bench.py --replicas $r --steps 2 --warmup 1 --no-cpu-baseline > $OUT/b$r.json 2>$OUT/b$r.err
  python -c "import json; d=json.loads(open('$OUT/b$r.json').read().strip().splitlines()[-1]); print($r, round(d['value']/1e6,1), round(d['ms_per_step'],1), round(d['roofline']['kernel_ms'],1))" >> $OUT/sweep.txt 2>&1
done
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section WarpStateStats --section LaunchStats --section SchedulerStats --clock-control none -k regex:sched_kernel --launch-skip 1 --launch-count 1 -o $OUT/mem1184 -f python bench.py --replicas 1184 --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu.log 2>&1
echo ncu $?
cat $OUT/time_case.txt $OUT/sweep.txt
