OUT=gpurun_out/$1; mkdir -p $OUT
for round in 1 2; do for v in 0 1; do
  PB_POOL_ROUND=$v timeout 600 python bench.py --replicas 2368 --steps 2 --warmup 1 --no-cpu-baseline > $OUT/r$v$round.json 2>$OUT/r$v$round.err
  python -c "import json; d=json.loads(open('$OUT/r$v$round.json').read().strip().splitlines()[-1]); print('round=$v run$round', round(d['value']/1e6,1), 'M/s engine', round(d['roofline']['kernel_ms'],1))"
done; done
