OUT=gpurun_out/r2w; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], d['clocks'])"
PB_SLOW=1 timeout 1200 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "c4_full_fcfs" > $OUT/pytest_c4full.log 2>&1; echo "c4 full test exit $?"; tail -2 $OUT/pytest_c4full.log
