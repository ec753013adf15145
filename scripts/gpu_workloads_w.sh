OUT=gpurun_out/$1; mkdir -p $OUT
for w in c1 c5; do for m in 8 12 16; do
  PB_MAX_WARPS_PER_SM=$m timeout 900 python bench.py --workload $w --replicas ${2:-9472} --steps 2 --warmup 1 --no-cpu-baseline > $OUT/b_${w}_$m.json 2> $OUT/b_${w}_$m.err
  python -c "import json; d=json.loads(open('$OUT/b_${w}_$m.json').read().strip().splitlines()[-1]); print('$w w$m', round(d['value']/1e6,1), 'M/s step', round(d['ms_per_step'],1))"
done; done
