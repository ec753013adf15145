# round 2: full GPU suite, instance-parallel parity + timings, sanitizers, default bench
OUT=gpurun_out/r2a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
PB_PDES_DEBUG=1 timeout 600 python scripts/pdes_check.py parity > $OUT/pdes_parity.txt 2>&1; echo "pdes parity exit $?"; tail -1 $OUT/pdes_parity.txt
timeout 600 python scripts/pdes_check.py time c2_pascal c3_l8_pascal c3_l8_fcfs c3_l8_nonadaptive c4s_pascal c4s_fcfs > $OUT/pdes_times.txt 2>&1; cat $OUT/pdes_times.txt | cut -c1-300
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  timeout 900 $CS --tool $tool --print-limit 30 --error-exitcode 9 python scripts/sanitize_cases.py > $OUT/san_${tool}.log 2>&1
  echo "$tool exit $?" | tee -a $OUT/san_summary.txt; tail -2 $OUT/san_${tool}.log
done
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"; tail -c 3000 $OUT/bench.json
