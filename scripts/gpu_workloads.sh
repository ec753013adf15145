# Bench lines for the other workloads (C1 and the C5 replica-sweep slice).
OUT=gpurun_out/$1; mkdir -p $OUT
for w in c1 c5; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  echo "$w exit $?"; python -c "import json; d=json.loads(open('$OUT/bench_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']/1e6,1), 'M/s step', round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']/1e6,1), 'frac', d['roofline']['frac'], 'cpu', d['cpu_baseline'] and d['cpu_baseline']['value'], d.get('parity_vs_cpu_ref',{}) and d['parity_vs_cpu_ref']['bit_exact'])"
done
