# Parity tests + a short replica sweep of bench.py.
#   bash scripts/gpu_check.sh LABEL "REPLICAS..." [skip-tests]
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
if [ "${3:-}" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu.log; tail -4 $OUT/pytest_gpu.log
fi
for spec in $2; do
  r=${spec%%:*}; w=${spec#*:}; [ "$w" = "$spec" ] && w=""
  if [ -n "$w" ]; then export PB_WARPS_PER_SM=$w; else unset PB_WARPS_PER_SM; fi
  timeout 300 python bench.py --replicas $r --steps 2 --warmup 1 --no-cpu-baseline > $OUT/b$spec.json 2>$OUT/b$spec.err
  python -c "import json; d=json.loads(open('$OUT/b$spec.json').read().strip().splitlines()[-1]); print('$spec', round(d['value']/1e6,1), 'M/s step', round(d['ms_per_step'],1), 'engine', round(d['roofline']['kernel_ms'],1))" 2>&1 | tail -1
done
unset PB_WARPS_PER_SM
python scripts/time_case.py c2_pascal 1
