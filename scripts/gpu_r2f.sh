# exact-seq PDES with the parallel merge: parity, timings, sanitizers, div_by A/B
OUT=gpurun_out/r2f; mkdir -p $OUT
PB_PDES_DEBUG=1 timeout 600 python scripts/pdes_check.py parity > $OUT/pdes_parity.txt 2>&1; echo "pdes parity exit $?"; grep -E "BAD|declined|parity:" $OUT/pdes_parity.txt | tail -8
PB_PDES_DEBUG=1 timeout 900 python scripts/pdes_check.py time c2_pascal c3_l8_pascal c3_l8_nonadaptive c3_l16_pascal c3_l8_fcfs c4s_pascal c4s_fcfs > $OUT/pdes_times.txt 2>&1; grep case $OUT/pdes_times.txt | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['case'], d['instance_parallel'], round(d['derive_ms']), round(d['engine_ms']), round(d['total_ms']))"
timeout 1500 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "xlarge or instance_parallel" > $OUT/pytest_xl.log 2>&1; echo "pytest xl exit $?"; tail -3 $OUT/pytest_xl.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 10 --error-exitcode 9 python scripts/sanitize_cases.py > $OUT/san_${tool}.log 2>&1
  echo "$tool exit $?"; tail -1 $OUT/san_${tool}.log
done
bash scripts/gpu_ab.sh r2f/ab build/ab/libA_base.so 2368
