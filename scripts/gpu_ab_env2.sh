# A/B of an env knob in one session: bash scripts/gpu_ab_env2.sh LABEL VAR VAL_A VAL_B REPS [WORKLOAD]
OUT=gpurun_out/$1; mkdir -p $OUT
for round in 1 2; do for v in $3 $4; do
  env $2=$v timeout 600 python bench.py --workload ${6:-c2} --replicas $5 --steps 2 --warmup 1 --no-cpu-baseline > $OUT/$v$round.json 2>$OUT/$v$round.err
  python -c "import json; d=json.loads(open('$OUT/$v$round.json').read().strip().splitlines()[-1]); print('$2=$v run$round', round(d['value']/1e6,1), 'M/s engine', round(d['roofline']['kernel_ms'],1))"
done; done
