# A/B of two builds of libpascal.so in one session: bash scripts/gpu_ab.sh LABEL ALT_SO REPS
OUT=gpurun_out/$1; mkdir -p $OUT
L=paper_2602_11530_b200/libpascal.so
cp $L /tmp/libB.so
for round in 1 2; do
  for v in A B; do
    if [ $v = A ]; then cp $2 $L; else cp /tmp/libB.so $L; fi
    timeout 600 python bench.py --workload ${4:-c2} --replicas ${3:-2368} --steps 2 --warmup 1 --no-cpu-baseline > $OUT/$v$round.json 2>$OUT/$v$round.err
    python -c "import json; d=json.loads(open('$OUT/$v$round.json').read().strip().splitlines()[-1]); print('$v$round', round(d['value']/1e6,1), 'M/s engine', round(d['roofline']['kernel_ms'],1))"
  done
done
cp /tmp/libB.so $L
