# replicas per GPU: 4 vs 8 per warp (work-stealing tail amortisation)
OUT=gpurun_out/r2reps; mkdir -p $OUT
for round in 1 2; do
  for r in 4736 9472; do
    timeout 900 python bench.py --replicas $r --steps 2 --warmup 1 --no-cpu-baseline > $OUT/r$r.$round.json 2> $OUT/r$r.$round.err
    python -c "import json; d=json.loads(open('$OUT/r$r.$round.json').read().strip().splitlines()[-1]); print('$r', round(d['value']/1e6,1), 'M/s step', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']/1e6,1))"
  done
done
