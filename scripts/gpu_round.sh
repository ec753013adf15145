#!/usr/bin/env bash
# One GPU session: parity tests, bench lines, launch list and one ncu --set full
# capture of the policy-run sched_kernel. Usage (from the repo root, on the box):
#   bash scripts/gpu_round.sh LABEL [REPLICAS_FOR_NCU] [skip-tests]
set -u
LABEL=${1:-r1}
NREP=${2:-296}
OUT=gpurun_out/$LABEL
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt" 2>&1
if [ "${3:-}" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
  tail -3 "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.log"
  tail -2 "$OUT/smoke.log"
fi
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?"; tail -c 3000 "$OUT/bench.json"
for r in ${BENCH_EXTRA:-}; do
  timeout 600 python bench.py --replicas "$r" --no-cpu-baseline > "$OUT/bench_r$r.json" 2> "$OUT/bench_r$r.err"
  echo "bench r=$r exit $?"; python -c "import json,sys; d=json.loads(open('$OUT/bench_r$r.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > "$OUT/launches_bench.log" 2>&1
echo "ncu launches exit $?"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:sched_kernel --launch-skip 1 --launch-count 1 -o "$OUT/prof" -f \
  python bench.py --replicas "$NREP" --steps 1 --warmup 0 --no-cpu-baseline \
  > "$OUT/ncu_full.log" 2>&1
echo "ncu full exit $?"; tail -5 "$OUT/ncu_full.log"
