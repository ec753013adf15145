# final tree: A/B of the last gather tweak, full GPU suite, smoke, bench line
bash scripts/gpu_abn.sh r2y 2368 build/ab/libN_check.so build/ab/libP2_dm.so
OUT=gpurun_out/r2y; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], d['clocks'])"
