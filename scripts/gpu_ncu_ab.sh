# instruction / issue counters of the policy-run sched_kernel for several builds:
#   bash scripts/gpu_ncu_ab.sh LABEL REPS SO1 SO2 ...
OUT=gpurun_out/$1; mkdir -p $OUT; REPS=$2; shift 2
L=paper_2602_11530_b200/libpascal.so
cp $L /tmp/libcur.so
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__average_warp_latency_issue_stalled_no_instruction.ratio,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum
for so in "$@"; do
  v=$(basename $so .so)
  cp $so $L
  timeout 900 ncu --metrics $M --clock-control none -k regex:sched_kernel --launch-skip 1 --launch-count 1 --csv \
    python bench.py --replicas $REPS --steps 1 --warmup 0 --no-cpu-baseline > $OUT/$v.csv 2> $OUT/$v.err
  python - "$OUT/$v.csv" "$v" <<'PY'
import csv, sys
rows = [r for r in csv.reader([l for l in open(sys.argv[1]) if l.startswith(chr(34))]) if len(r) > 10]
hdr = rows[0]; i_n = hdr.index("Metric Name"); i_v = hdr.index("Metric Value")
print(sys.argv[2], {r[i_n].replace("smsp__average_warps_issue_stalled_", "st_").replace("_per_issue_active.ratio", ""): r[i_v] for r in rows[1:]})
PY
done
cp /tmp/libcur.so $L
