# C5 thrash points (k < 3, capacity 0.5) as single pascal_run calls on the GPU
OUT=gpurun_out/$1; mkdir -p $OUT
for c in c5_s0_k0_fcfs c5_s0_k1_pascal c5_s0_k0_pascal c5_s0_k0_nomig c5_s1_k0_pascal; do
  timeout 600 python scripts/single_runs.py $OUT/thrash.jsonl $c >> $OUT/thrash.log 2>&1; echo "$c exit $?"
done
cut -c1-330 $OUT/thrash.jsonl
