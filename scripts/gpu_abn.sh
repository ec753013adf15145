# A/B/... of several builds in one session: bash scripts/gpu_abn.sh LABEL REPS SO1 SO2 ...
OUT=gpurun_out/$1; mkdir -p $OUT; REPS=$2; shift 2
L=paper_2602_11530_b200/libpascal.so
cp $L /tmp/libcur.so
for round in 1 2; do
  for so in "$@"; do
    v=$(basename $so .so)
    cp $so $L
    timeout 600 python bench.py --workload ${WL:-c2} --replicas $REPS --steps 2 --warmup 1 --no-cpu-baseline > $OUT/$v$round.json 2>$OUT/$v$round.err
    python -c "import json; d=json.loads(open('$OUT/$v$round.json').read().strip().splitlines()[-1]); print('$v$round', round(d['value']/1e6,1), 'M/s engine', round(d['roofline']['kernel_ms'],1), 'e2e', round(d['e2e']['value']/1e6,1))"
  done
done
cp /tmp/libcur.so $L
