# Round-2 evidence: default bench line (+ CPU baseline), the reference arm,
# launch list, DRAM bytes of the default launch, other workloads, single-run
# latency of the drop-in path (C3 / C4), ncu --set full at 1,184 replicas.
#   bash scripts/gpu_final_r2.sh LABEL
L=$1
OUT=gpurun_out/$L; mkdir -p $OUT
bash scripts/gpu_bench_default.sh $L | grep -v "^{"
python -c "import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])"
for w in c5 c1; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  echo "bench $w exit $?"; python -c "import json; d=json.loads(open('$OUT/bench_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])"
done
timeout 1500 python scripts/single_runs.py $OUT/single.jsonl c3_l8_pascal:cpu c3_l8_fcfs:cpu c4s_pascal:cpu c3_l16_pascal c3x_l8_pascal c3_l8_nonadaptive > $OUT/single.log 2>&1
echo "single exit $?"; cut -c1-400 $OUT/single.jsonl
bash scripts/gpu_ncu_full.sh $L 1184
