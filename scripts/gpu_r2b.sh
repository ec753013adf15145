# round 2: new unit-parity / caller / tpot / multi-device tests, PDES decline reasons, sanitizers
OUT=gpurun_out/r2b; mkdir -p $OUT
PB_PDES_DEBUG=1 timeout 300 python scripts/pdes_check.py time c3_l8_nonadaptive c3_l16_pascal c3_l16_nonadaptive > $OUT/pdes_debug.txt 2>&1; grep -v "^\[pdes\] .*replica [1-9]" $OUT/pdes_debug.txt | cut -c1-400 | head -30
timeout 900 python -m pytest tests/test_unit_probe.py tests/test_callers.py tests/test_tpot_gpu.py tests/test_multi_device.py -q -m gpu -x > $OUT/pytest_new.log 2>&1; echo "pytest new exit $?"; tail -30 $OUT/pytest_new.log
PB_PDES_DEBUG=1 timeout 600 python scripts/pdes_check.py parity > $OUT/pdes_parity.txt 2>&1; echo "pdes parity exit $?"; tail -1 $OUT/pdes_parity.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in synccheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 10 --error-exitcode 9 python scripts/sanitize_cases.py > $OUT/san_${tool}.log 2>&1
  echo "$tool exit $?"; tail -2 $OUT/san_${tool}.log
done
