# C4 at its stated size (1 M requests, 64 instances): GPU pascal_run timing
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 3000 python scripts/single_runs.py $OUT/c4full.jsonl c4_full_fcfs c4_full_pascal > $OUT/c4full.log 2>&1
echo "c4full exit $?"; cat $OUT/c4full.jsonl; tail -3 $OUT/c4full.log
